// pv4: output_aligned for every G from a per-warp TMA ring with a lean
// lane map.  Included by akv_pv.cu.
//
// Every warp owns a balanced contiguous range of (unit, page) items and streams each
// page as 32-row stages through a private NS-slot ring: lane 0 issues one
// cp.async.bulk of the stage's V head rows (4 KB, token-major; uniform tiers add the
// stage's mid / low rows), G 128 B copies of the heads' p_t for those rows and, with a
// page's first stage, the page's selection / fetch-plan words (akv_softmax_select).
// Lane = (row half, 8-channel group): lanes 0-15 walk rows 0-15 of the stage, lanes
// 16-31 rows 16-31, each lane over channels 8cg .. 8cg+7, so per row a lane does one
// LDS.64 of head bytes, 4 PRMT (T8 words, midpoint fill HB:160-179), 8 conversions and
// 4 FFMA2 per q-head; a lane's accumulators are 8 fp32 per head (G = 4: 32, the whole
// group in one pass).  Selected rows (D6) and rows past the length get p = 0 in the
// stage's p block.  Rows in the union fetch plan (rare) go through the out-of-line
// per-element rule of pv3 (v_row_generic: unknown target -> T16,
// p_t = 0 -> T8 (D5), element / row strategy (D4 / D7)).  The page partial goes to
// o_partial[h][page]; akv_combine adds o_est and the partials in a fixed order.

namespace akv {

template <int G, bool UNIFORM>
struct Pv4Shape {
  static constexpr int R = 32;                      // rows per stage
  static constexpr int HEAD = R * D;                // 4 KB
  static constexpr int NIB = UNIFORM ? R * (D / 2) : 0;
  static constexpr int PB = G * R * 4;              // p block [G][R]
  static constexpr int SLOT = HEAD + 2 * NIB + PB;
  static constexpr int META = G * 96;               // per page: sel[G][8] words, need[G][2][8] words
  static constexpr int NS = 3;
  static constexpr int WARPS = 4;
  static constexpr int PER_WARP = (NS * SLOT + 2 * META + NS * 8 + 127) & ~127;
  static constexpr int SMEM = WARPS * PER_WARP;
  static constexpr int MINB = G <= 2 ? 4 : (G == 4 ? 3 : 2);
};

template <int G, bool UNIFORM>
__device__ __forceinline__ void pv4_issue(uint8_t* slot, uint8_t* meta, uint64_t* bar, const PvCursor& c,
                                          const akv_store_t& s, const akv_step_t& st, int cap) {
  using S = Pv4Shape<G, UNIFORM>;
  const uint8_t* vb = s.v_pool + c.pid * PAGE;
  const int r0 = c.sub * S::R;
  const int capw = cap >> 5;
  const bool first = c.sub == 0;
  mbar_arrive_expect_tx(bar, S::HEAD + 2 * S::NIB + S::PB + (first && !UNIFORM ? S::META : 0));
  bulk_g2s(slot, vb + r0 * D, S::HEAD, bar);
  if (UNIFORM) {
    bulk_g2s(slot + S::HEAD, vb + MID + r0 * (D / 2), S::NIB, bar);
    bulk_g2s(slot + S::HEAD + S::NIB, vb + LOW + r0 * (D / 2), S::NIB, bar);
  }
#pragma unroll
  for (int j = 0; j < G; ++j)
    bulk_g2s(slot + S::HEAD + 2 * S::NIB + j * S::R * 4, st.probs + ((size_t)c.u * G + j) * cap + (size_t)c.pg * P + r0,
             S::R * 4, bar);
  if (first && !UNIFORM) {
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const size_t h = (size_t)c.u * G + j;
      bulk_g2s(meta + j * 32, st.sel_bits + h * capw + c.pg * 8, 32, bar);
      const uint32_t* nb = st.need_bits + h * 2 * capw + c.pg * 8;
      bulk_g2s(meta + G * 32 + j * 64, nb, 32, bar);
      bulk_g2s(meta + G * 32 + j * 64 + 32, nb + capw, 32, bar);
    }
  }
}

// T8 words of 8 head bytes (channels 8cg .. +7) -> 4 float2.
__device__ __forceinline__ void t8_f2(const uint2 hv, float2 (&f)[4]) {
  const uint32_t c80 = 0x80808080u;
  f[0] = half2_bits_to_float2(prmt(hv.x, c80, 0x1404));
  f[1] = half2_bits_to_float2(prmt(hv.x, c80, 0x3424));
  f[2] = half2_bits_to_float2(prmt(hv.y, c80, 0x1404));
  f[3] = half2_bits_to_float2(prmt(hv.y, c80, 0x3424));
}

template <int G>
struct Pv4Gen {  // contributions of the out-of-line row path (returned by value: the caller's
  float2 acc[G][4];  // accumulators stay in registers)
  int adj[G][3];
};

// One aligned row in the union fetch plan, this lane's 8 channels, every head: the per-head
// mode (selected -> skip, not in the head's plan -> T8, row strategy -> row tier, element
// strategy -> per-element rule D4) on the fetched nibbles.  Out of line (rare).
// selm / needm: the page's selection [G][8] and fetch-plan [G][2][8] words (shared memory);
// pb: the stage's p block [G][32].
template <int G, bool EXPORT>
__device__ __noinline__ Pv4Gen<G> pv4_row_generic(uint2 hv, int row, int rr, const uint8_t* vb, const float* pb,
                                                  const uint32_t* selm, const uint32_t* needm, int u, int pg, int cap,
                                                  akv_cfg_t cfg, const int32_t* targets, uint8_t* v_tiers) {
  // (the step struct is not passed by pointer: taking its address would move the kernel's
  // parameter copy to local memory)
  const int lane = threadIdx.x & 31, cg = lane & 15;
  const int chk = row >> 5, bit = row & 31;
  Pv4Gen<G> out;
#pragma unroll
  for (int j = 0; j < G; ++j) {
    out.adj[j][0] = out.adj[j][1] = out.adj[j][2] = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) out.acc[j][q] = make_float2(0.f, 0.f);
  }
  // the union plan decides what is fetched (one 4 B word per nibble plane for this lane)
  uint32_t um = 0u, ul = 0u;
#pragma unroll
  for (int j = 0; j < G; ++j) {
    um |= needm[j * 16 + chk];
    ul |= needm[j * 16 + 8 + chk];
  }
  uint32_t mw = 0u, lw = 0u;
  if ((um >> bit) & 1u) mw = __ldg(reinterpret_cast<const uint32_t*>(vb + MID + row * (D / 2) + cg * 4));
  if ((ul >> bit) & 1u) lw = __ldg(reinterpret_cast<const uint32_t*>(vb + LOW + row * (D / 2) + cg * 4));
#pragma unroll
  for (int j = 0; j < G; ++j) {
    const size_t h = (size_t)u * G + j;
    const float pv = pb[j * 32 + rr];
    uint8_t* vt = EXPORT && v_tiers ? v_tiers + (h * cap + (size_t)pg * P + row) * D + cg * 8 : nullptr;
    int mode;  // 0 skip, 1 element, 8/12/16 tier
    if ((selm[j * 8 + chk] >> bit) & 1u) {
      mode = 0;
    } else if (!((needm[j * 16 + chk] >> bit) & 1u)) {
      mode = 8;
    } else if (cfg.strategy == 1) {
      mode = ((needm[j * 16 + 8 + chk] >> bit) & 1u) ? 16 : 12;
    } else {
      mode = 1;
    }
    uint32_t w[4];
    uint32_t cds[2] = {0u, 0u};
    if (mode == 0) {
      if (EXPORT && vt) *reinterpret_cast<uint2*>(vt) = make_uint2(0x10101010u, 0x10101010u);
      continue;
    }
    if (mode == 8) {
      const uint32_t c80 = 0x80808080u;
      w[0] = prmt(hv.x, c80, 0x1404);
      w[1] = prmt(hv.x, c80, 0x3424);
      w[2] = prmt(hv.y, c80, 0x1404);
      w[3] = prmt(hv.y, c80, 0x3424);
      cds[0] = cds[1] = 0x08080808u;
    } else if (mode != 1) {
      const TierMask tm = tier_mask(mode);
      assemble8(hv.x, hv.y, bsel(tm.mk, mw, 0x88888888u), bsel(tm.lk, lw, tm.lf), w);
      out.adj[j][0] -= 8;
      out.adj[j][mode == 12 ? 1 : 2] += 8;
      cds[0] = cds[1] = (uint32_t)mode * 0x01010101u;
    } else {
      assemble8(hv.x, hv.y, mw, lw, w);
      const int ep = pv > 0.f ? floor_log2f(pv) : -30000;
      const int4* tp = reinterpret_cast<const int4*>(targets + h * D + cg * 8);
      const int4 t0 = tp[0], t1 = tp[1];
      const int tg[8] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w};
      const uint32_t hb[2] = {hv.x, hv.y};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int g = tg[e] == AKV_TARGET_UNKNOWN ? -(1 << 20) : 17 + tg[e] - cfg.margin_bits;
        const uint32_t hbyte = (hb[e >> 2] >> (8 * (e & 3))) & 0xFFu;
        const int E = max((int)((hbyte >> 2) & 31u), 1) + ep;
        const bool km = E > g, kl = E > g + 4;
        const int sh = 16 * (e & 1);
        uint32_t w16 = (w[e >> 1] >> sh) & 0xFFFFu;
        w16 = kl ? w16 : (km ? ((w16 & 0xFFF0u) | 0x8u) : ((w16 & 0xFF00u) | 0x80u));
        w[e >> 1] = (w[e >> 1] & ~(0xFFFFu << sh)) | (w16 << sh);
        out.adj[j][0] -= km ? 1 : 0;
        out.adj[j][1] += (km && !kl) ? 1 : 0;
        out.adj[j][2] += kl ? 1 : 0;
        cds[e >> 2] |= (kl ? 16u : (km ? 12u : 8u)) << (8 * (e & 3));
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) out.acc[j][k] = ffma2_scalar(half2_bits_to_float2(w[k]), pv, out.acc[j][k]);
    if (EXPORT && vt) *reinterpret_cast<uint2*>(vt) = make_uint2(cds[0], cds[1]);
  }
  return out;
}

template <int G, bool TRUNC, bool EXPORT, bool UNIFORM>
__global__ void __launch_bounds__(32 * Pv4Shape<G, UNIFORM>::WARPS, Pv4Shape<G, UNIFORM>::MINB)
    pv4_kernel(akv_store_t s, akv_cfg_t cfg, akv_step_t st, int cap, int npg_max) {
  using S = Pv4Shape<G, UNIFORM>;
  constexpr int NS = S::NS, R = S::R;
  extern __shared__ __align__(128) uint8_t pv4_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = lane >> 4, cg = lane & 15;
  uint8_t* ring = pv4_smem + warp * S::PER_WARP;
  uint8_t* metab = ring + NS * S::SLOT;
  uint64_t* full = reinterpret_cast<uint64_t*>(metab + 2 * S::META);
  if (lane == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&full[i], 1);
    mbar_fence_init();
  }
  __syncwarp();
  pdl_trigger();
  pdl_wait();
  const int uni = TRUNC ? 16 : cfg.force_tier;
  uint32_t tkm = 0xFFFFFFFFu, tf = 0u;
  if (TRUNC) {
    const int kb = cfg.trunc_bits - 6;
    const uint32_t km = (0xFFFFu << (10 - kb)) & 0xFFFFu;
    const uint32_t fill = kb < 10 ? (1u << (9 - kb)) : 0u;
    tkm = km | (km << 16);
    tf = fill | (fill << 16);
  }
  const long long total = (long long)s.n_units * npg_max;
  const long long nw = (long long)gridDim.x * S::WARPS, gw = (long long)blockIdx.x * S::WARPS + warp;
  const long long i0 = total * gw / nw, i1 = total * (gw + 1) / nw;

  PvCursor ic, cc;  // issue / consume cursors over (unit, page, stage)
  ic.item = i0;
  ic.pass = 0;
  ic.u = (int)(i0 / npg_max);
  ic.pg = (int)(i0 % npg_max);
  ic.up.u = -1;
  ic.up.n = 0;
  ic.npage = 0;
  bool iv = pv_cursor_seek<R>(ic, i1, s, npg_max, 1);
  cc = ic;
  bool cv = iv;
  int kiss = 0;
  for (; kiss < NS - 1 && iv; ++kiss) {
    if (lane == 0)
      pv4_issue<G, UNIFORM>(ring + (kiss % NS) * S::SLOT, metab + (ic.npage & 1) * S::META, &full[kiss % NS], ic, s,
                            st, cap);
    iv = pv_cursor_next<R>(ic, i1, s, npg_max, 1);
  }

  float2 acc[G][4];
  int adj[G][3], base[G];
  const uint8_t* vb = nullptr;
  long long vbytes = 0;  // physical V bytes of the current page (lane 0)
  for (int k = 0; cv; ++k) {
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    // the page meta is double-buffered: page N+2's first stage waits until page N is consumed
    if (iv && (ic.sub != 0 || ic.npage - cc.npage < 2)) {
      if (lane == 0)
        pv4_issue<G, UNIFORM>(ring + (kiss % NS) * S::SLOT, metab + (ic.npage & 1) * S::META, &full[kiss % NS], ic,
                              s, st, cap);
      ++kiss;
      iv = pv_cursor_next<R>(ic, i1, s, npg_max, 1);
    }
    const int slot = k % NS;
    mbar_wait(&full[slot], (uint32_t)(k / NS) & 1u);
    uint8_t* sd = ring + slot * S::SLOT;
    float* pb = reinterpret_cast<float*>(sd + S::HEAD + 2 * S::NIB);
    const uint32_t* md = reinterpret_cast<const uint32_t*>(metab + (cc.npage & 1) * S::META);
    const uint32_t* selm = md;           // [G][8]
    const uint32_t* needm = md + G * 8;  // [G][2][8]
    if (cc.sub == 0) {
#pragma unroll
      for (int j = 0; j < G; ++j) {
        adj[j][0] = adj[j][1] = adj[j][2] = 0;
        base[j] = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[j][q] = make_float2(0.f, 0.f);
      }
      vb = s.v_pool + cc.pid * PAGE;
      vbytes = 0;
    }
    const int r0 = cc.sub * R;
    const int nvs = min(R, cc.rows - r0);  // valid rows of this stage
    // this stage's 32-row chunk: selection and union fetch-plan words
    const int chk = r0 >> 5;
    uint32_t selw[G], um = 0u;
#pragma unroll
    for (int j = 0; j < G; ++j) {
      selw[j] = UNIFORM ? 0u : selm[j * 8 + chk];
      if (!UNIFORM) um |= needm[j * 16 + chk] | needm[j * 16 + 8 + chk];
    }
    const uint32_t vmask = nvs >= 32 ? 0xFFFFFFFFu : ((1u << nvs) - 1u);
    um &= vmask;
    if (UNIFORM) {
      vbytes += (long long)nvs * (D + (uni >= 12 ? D / 2 : 0) + (uni >= 16 ? D / 2 : 0));
    } else {
      uint32_t wm = 0u, wl = 0u;  // the union plan's nibble rows of this chunk
#pragma unroll
      for (int j = 0; j < G; ++j) {
        wm |= needm[j * 16 + chk];
        wl |= needm[j * 16 + 8 + chk];
      }
      vbytes += (long long)nvs * D + (long long)(__popc(wm & vmask) + __popc(wl & vmask)) * (D / 2);
    }
    // p = 0 for selected rows (D6: their T16 term is o_est) and rows past the length; counts
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const bool zero = !((vmask >> lane) & 1u) || ((selw[j] >> lane) & 1u);
      if (zero) pb[j * R + lane] = 0.f;
      base[j] += nvs - __popc(selw[j] & vmask);
    }
    __syncwarp();

    // rows of this lane: r = 16 * half + i, i = 0..15
    const uint8_t* hrow = sd + (16 * half) * D + cg * 8;
    if (UNIFORM) {
      const TierMask tm = tier_mask(uni);
      const uint8_t* mrow = sd + S::HEAD + (16 * half) * (D / 2) + cg * 4;
#pragma unroll 4
      for (int i = 0; i < 16; ++i) {
        const uint2 hv = *reinterpret_cast<const uint2*>(hrow + i * D);
        const uint32_t mw = *reinterpret_cast<const uint32_t*>(mrow + i * (D / 2));
        const uint32_t lw = *reinterpret_cast<const uint32_t*>(mrow + S::NIB + i * (D / 2));
        uint32_t w[4];
        assemble8(hv.x, hv.y, bsel(tm.mk, mw, 0x88888888u), bsel(tm.lk, lw, tm.lf), w);
        if (TRUNC) {
#pragma unroll
          for (int q = 0; q < 4; ++q) w[q] = (w[q] & tkm) | tf;
        }
        float2 f[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) f[q] = half2_bits_to_float2(w[q]);
#pragma unroll
        for (int j = 0; j < G; ++j) {
          const float pv = pb[j * R + 16 * half + i];
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[j][q] = ffma2_scalar(f[q], pv, acc[j][q]);
        }
        if (EXPORT && st.v_tiers && 16 * half + i < nvs) {
          const uint32_t cd = (uint32_t)uni * 0x01010101u;
#pragma unroll
          for (int j = 0; j < G; ++j)
            *reinterpret_cast<uint2*>(st.v_tiers +
                                      (((size_t)cc.u * G + j) * cap + (size_t)cc.pg * P + r0 + 16 * half + i) * D +
                                      cg * 8) = make_uint2(cd, cd);
        }
      }
    } else if (um == 0u && !EXPORT) {
      // fast stage: every row T8 (or p = 0)
#pragma unroll 4
      for (int i = 0; i < 16; i += 4) {
        float4 p4[G];
#pragma unroll
        for (int j = 0; j < G; ++j) p4[j] = *reinterpret_cast<const float4*>(pb + j * R + 16 * half + i);
#pragma unroll
        for (int ii = 0; ii < 4; ++ii) {
          const uint2 hv = *reinterpret_cast<const uint2*>(hrow + (i + ii) * D);
          float2 f[4];
          t8_f2(hv, f);
#pragma unroll
          for (int j = 0; j < G; ++j) {
            const float pv = ii == 0 ? p4[j].x : (ii == 1 ? p4[j].y : (ii == 2 ? p4[j].z : p4[j].w));
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[j][q] = ffma2_scalar(f[q], pv, acc[j][q]);
          }
        }
      }
    } else {
      // rows in the union fetch plan through the per-element rule; the rest T8 (row pairs of
      // the two halves share the decision so the warp stays converged)
#pragma unroll 1
      for (int i = 0; i < 16; ++i) {
        const int rr = 16 * half + i, row = r0 + rr;
        const uint2 hv = *reinterpret_cast<const uint2*>(hrow + i * D);
        const bool gen = ((um >> i) & 1u) || ((um >> (16 + i)) & 1u) || EXPORT;
        if (!gen) {
          float2 f[4];
          t8_f2(hv, f);
#pragma unroll
          for (int j = 0; j < G; ++j) {
            const float pv = pb[j * R + rr];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[j][q] = ffma2_scalar(f[q], pv, acc[j][q]);
          }
        } else if (rr < nvs) {
          const Pv4Gen<G> g = pv4_row_generic<G, EXPORT>(hv, row, rr, vb, pb, selm, needm, cc.u, cc.pg, cap, cfg, st.targets,
                                                               st.v_tiers);
#pragma unroll
          for (int j = 0; j < G; ++j) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              acc[j][q].x += g.acc[j][q].x;
              acc[j][q].y += g.acc[j][q].y;
            }
            adj[j][0] += g.adj[j][0];
            adj[j][1] += g.adj[j][1];
            adj[j][2] += g.adj[j][2];
          }
        }
      }
    }

    if (cc.sub + 1 == cc.nsub) {
      if (lane == 0)
        atomicAdd(reinterpret_cast<unsigned long long*>(st.unit_bytes + (size_t)cc.u * 4 + 1),
                  (unsigned long long)vbytes);
      // page end: fold the two row halves, lanes 0..15 write 8 channels per head; counters
#pragma unroll
      for (int j = 0; j < G; ++j) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          acc[j][q].x += __shfl_xor_sync(0xFFFFFFFFu, acc[j][q].x, 16);
          acc[j][q].y += __shfl_xor_sync(0xFFFFFFFFu, acc[j][q].y, 16);
        }
        const size_t h = (size_t)cc.u * G + j;
        if (half == 0) {
          float4* dst = reinterpret_cast<float4*>(st.o_partial + (h * (cap / P) + cc.pg) * D + cg * 8);
          dst[0] = make_float4(acc[j][0].x, acc[j][0].y, acc[j][1].x, acc[j][1].y);
          dst[1] = make_float4(acc[j][2].x, acc[j][2].y, acc[j][3].x, acc[j][3].y);
        }
        const int a = warp_sum_i(adj[j][0]), b1 = warp_sum_i(adj[j][1]), c2 = warp_sum_i(adj[j][2]);
        if (lane == 0) {
          unsigned long long* ct = reinterpret_cast<unsigned long long*>(st.counters + h * 8 + 3);
          long long t8 = a, t12 = b1, t16 = c2;
          const long long bs = (long long)base[j] * D;
          if (!UNIFORM || uni == 8) t8 += bs;
          else if (uni == 12) t12 += bs;
          else t16 += bs;
          if (t8) atomicAdd(ct + 0, (unsigned long long)t8);
          if (t12) atomicAdd(ct + 1, (unsigned long long)t12);
          if (t16) atomicAdd(ct + 2, (unsigned long long)t16);
        }
      }
    }
    cv = pv_cursor_next<R>(cc, i1, s, npg_max, 1);
  }
}

template <int G, bool TRUNC, bool EXPORT, bool UNIFORM>
static void launch_pv4_t(const akv_store_t& s, const akv_cfg_t& cfg, const akv_step_t& st, int max_len,
                         cudaStream_t stream) {
  using S = Pv4Shape<G, UNIFORM>;
  const int resident = resident_ctas<pv4_kernel<G, TRUNC, EXPORT, UNIFORM>>(32 * S::WARPS, S::SMEM);
  const int cap = s.max_pages * P;
  const int npg = (max_len + P - 1) / P;
  const long long items = (long long)s.n_units * npg;
  const int grid = balanced_grid(items, resident, S::WARPS);
  launch_pdl(PDL_PV, pv4_kernel<G, TRUNC, EXPORT, UNIFORM>, dim3(grid), dim3(32 * S::WARPS), (size_t)S::SMEM, stream, s, cfg,
             st, cap, npg);
}

}  // namespace akv
