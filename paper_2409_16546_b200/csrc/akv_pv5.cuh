// pv5: output_aligned, aligned serving mode, T8 rows on the tensor cores.
// Included by akv_pv.cu after akv_pv4.cuh (shares PvCursor, pv4_row_generic).
//
// For one (unit, page) the T8 part of the output is a small GEMM,
//   o_j[c] = sum_t p_jt * V8[t][c]          (V8 = head byte << 8 | 0x80, HB:160-179),
// which mma.sync m16n8k16 (fp16 in, fp32 accumulate) computes with
//   A[m][k] = V8[token k][channel(m)]  (16 channels x 16 tokens),
//   B[k][n] = p of token k for column n = (head n/2, hi if n even / lo if odd),
// p split as p * 2^14 = hi + lo, both fp16 (products exact in fp32; p and o keep ~22 bits),
// so one mma serves 4 q-heads (G = 8: two n-tiles).  The A fragments come straight from
// the TMA-staged head rows: a stage is 32 token rows x 128 B loaded by one
// cp.async.bulk.tensor.2d (UTMALDG, SWIZZLE_128B), and ldmatrix.trans on 16-bit
// (channel-pair) elements hands each lane the bytes (t, 2g), (t, 2g+1), (t+1, 2g),
// (t+1, 2g+1); two PRMT per register turn them into the T8 word pairs of channels 2g and
// 2g+1 (A rows g and g+8).  Selected rows (D6), rows past the length and rows in the union
// fetch plan get p = 0 in B; the plan rows run through the per-element rule on the CUDA
// cores (pv4_row_generic) into a per-warp shared buffer added at the page end.  Per-page
// partials go to o_partial; akv_combine adds o_est and the partials in a fixed order.

namespace akv {

template <int G>
struct Pv5Shape {
  static constexpr int R = 32;             // rows per stage
  static constexpr int HEAD = R * D;       // 4 KB, 1 KB aligned (SWIZZLE_128B)
  static constexpr int PB = G * R * 4;     // p block [G][R] per stage
  static constexpr int META = G * 96;      // per page: sel[G][8], need[G][2][8] words
  static constexpr int NS = 3;
  static constexpr int WARPS = 4;
  static constexpr int NT = G > 4 ? 2 : 1;  // n-tiles of 8 columns (4 heads each)
  // CTA: [WARPS x NS head tiles (4 KB, 1 KB aligned)] [WARPS x misc], misc per warp =
  // NS p blocks | 2 page metas | generic buffer [G][D] | NS mbarriers
  static constexpr int OFF_PB = 0;
  static constexpr int OFF_META = OFF_PB + NS * PB;
  static constexpr int OFF_GEN = OFF_META + 2 * META;
  static constexpr int OFF_BAR = OFF_GEN + G * D * 4;
  static constexpr int MISC = (OFF_BAR + NS * 8 + 15) & ~15;
  static constexpr int SMEM = WARPS * NS * HEAD + WARPS * MISC + 1024;  // + 1 KB alignment slack
  static constexpr int MINB = G <= 4 ? 3 : 2;
};

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(tm), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void ldsm_x4_trans(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}

__device__ __forceinline__ void mma_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                          uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// fp16 bits of x's hi (lo = false) or lo (lo = true) part, x = hi + lo.
__device__ __forceinline__ uint32_t hilo16(float x, bool lo) {
  const __half h = __float2half_rn(x);
  if (!lo) return __half_as_ushort(h);
  return __half_as_ushort(__float2half_rn(x - __half2float(h)));
}

template <int G>
__device__ __forceinline__ void pv5_issue(uint8_t* head, float* pblk, uint8_t* meta, uint64_t* bar, const PvCursor& c,
                                          const CUtensorMap* tm, const akv_step_t& st, int cap) {
  using S = Pv5Shape<G>;
  const int r0 = c.sub * S::R;
  const int capw = cap >> 5;
  const bool first = c.sub == 0;
  mbar_arrive_expect_tx(bar, S::HEAD + S::PB + (first ? S::META : 0));
  tma_load_2d(head, tm, 0, (int)(c.pid * 512 + r0), bar);  // V head rows of the stage (page = 512 rows of 128 B)
#pragma unroll
  for (int j = 0; j < G; ++j)
    bulk_g2s(pblk + j * S::R, st.probs + ((size_t)c.u * G + j) * cap + (size_t)c.pg * P + r0, S::R * 4, bar);
  if (first) {
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

template <int G>
struct Pv5Adj {
  int a[G][3];
};

// One row of the union fetch plan, this lane's 8 channels (8cg .. 8cg+7), every head: the
// per-head mode (selected -> skip, not in the head's plan -> T8, row strategy -> row tier,
// element strategy -> per-element rule D4, unknown target -> T16 SPEC.md:169) on the
// fetched nibbles, added into the warp's buffer gen[G][D].  Out of line and stateless
// (nothing but the tier-count adjustments comes back), so the caller's mma accumulators
// keep their registers.
template <int G>
__device__ __noinline__ Pv5Adj<G> pv5_row_rule(uint2 hv, int row, float* gen, const float* pb, int rr,
                                               const uint8_t* vb, const uint32_t* selm, const uint32_t* needm, int u,
                                               akv_cfg_t cfg, const int32_t* targets) {
  const int cg = threadIdx.x & 15;
  const int chk = row >> 5, bit = row & 31;
  Pv5Adj<G> out;
  uint32_t um = 0u, ul = 0u;
#pragma unroll
  for (int j = 0; j < G; ++j) {
    um |= needm[j * 16 + chk];
    ul |= needm[j * 16 + 8 + chk];
    out.a[j][0] = out.a[j][1] = out.a[j][2] = 0;
  }
  uint32_t mw = 0u, lw = 0u;
  if ((um >> bit) & 1u) mw = __ldg(reinterpret_cast<const uint32_t*>(vb + MID + row * (D / 2) + cg * 4));
  if ((ul >> bit) & 1u) lw = __ldg(reinterpret_cast<const uint32_t*>(vb + LOW + row * (D / 2) + cg * 4));
#pragma unroll 1
  for (int j = 0; j < G; ++j) {
    const float pv = pb[j * 32 + rr];
    int mode;  // 0 skip, 1 element, 8/12/16 tier
    if ((selm[j * 8 + chk] >> bit) & 1u) mode = 0;
    else if (!((needm[j * 16 + chk] >> bit) & 1u)) mode = 8;
    else if (cfg.strategy == 1) mode = ((needm[j * 16 + 8 + chk] >> bit) & 1u) ? 16 : 12;
    else mode = 1;
    if (mode == 0) continue;
    uint32_t w[4];
    if (mode == 8) {
      const uint32_t c80 = 0x80808080u;
      w[0] = prmt(hv.x, c80, 0x1404);
      w[1] = prmt(hv.x, c80, 0x3424);
      w[2] = prmt(hv.y, c80, 0x1404);
      w[3] = prmt(hv.y, c80, 0x3424);
    } else if (mode != 1) {
      const TierMask tm = tier_mask(mode);
      assemble8(hv.x, hv.y, bsel(tm.mk, mw, 0x88888888u), bsel(tm.lk, lw, tm.lf), w);
      out.a[j][0] -= 8;
      out.a[j][mode == 12 ? 1 : 2] += 8;
    } else {
      assemble8(hv.x, hv.y, mw, lw, w);
      const int ep = pv > 0.f ? floor_log2f(pv) : -30000;
      const int4* tp = reinterpret_cast<const int4*>(targets + ((size_t)u * G + j) * D + cg * 8);
      const int4 t0 = tp[0], t1 = tp[1];
      const int tg[8] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w};
      const uint32_t hb[2] = {hv.x, hv.y};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int gt = tg[e] == AKV_TARGET_UNKNOWN ? -(1 << 20) : 17 + tg[e] - cfg.margin_bits;
        const uint32_t hbyte = (hb[e >> 2] >> (8 * (e & 3))) & 0xFFu;
        const int E = max((int)((hbyte >> 2) & 31u), 1) + ep;
        const bool km = E > gt, kl = E > gt + 4;
        const int sh = 16 * (e & 1);
        uint32_t w16 = (w[e >> 1] >> sh) & 0xFFFFu;
        w16 = kl ? w16 : (km ? ((w16 & 0xFFF0u) | 0x8u) : ((w16 & 0xFF00u) | 0x80u));
        w[e >> 1] = (w[e >> 1] & ~(0xFFFFu << sh)) | (w16 << sh);
        out.a[j][0] -= km ? 1 : 0;
        out.a[j][1] += (km && !kl) ? 1 : 0;
        out.a[j][2] += kl ? 1 : 0;
      }
    }
    float* gj = gen + j * D + cg * 8;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = half2_bits_to_float2(w[k]);
      gj[2 * k] = fmaf(pv, f.x, gj[2 * k]);
      gj[2 * k + 1] = fmaf(pv, f.y, gj[2 * k + 1]);
    }
  }
  return out;
}

template <int G>
__global__ void __launch_bounds__(32 * Pv5Shape<G>::WARPS, Pv5Shape<G>::MINB)
    pv5_kernel(akv_store_t s, akv_cfg_t cfg, akv_step_t st, int cap, int npg_max, const __grid_constant__ CUtensorMap tmv) {
  using S = Pv5Shape<G>;
  constexpr int NS = S::NS, R = S::R, NT = S::NT;
  extern __shared__ __align__(1024) uint8_t pv5_raw[];
  uint8_t* pv5_smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(pv5_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;           // mma fragment coordinates
  uint8_t* heads = pv5_smem + warp * NS * S::HEAD;
  uint8_t* wbase = pv5_smem + S::WARPS * NS * S::HEAD + warp * S::MISC;
  float* pblks = reinterpret_cast<float*>(wbase + S::OFF_PB);
  uint8_t* metab = wbase + S::OFF_META;
  float* gen = reinterpret_cast<float*>(wbase + S::OFF_GEN);  // [G][D]
  uint64_t* full = reinterpret_cast<uint64_t*>(wbase + S::OFF_BAR);
  if (lane == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&full[i], 1);
    mbar_fence_init();
  }
  __syncwarp();
  pdl_trigger();
  pdl_wait();
  const long long total = (long long)s.n_units * npg_max;
  const long long nw = (long long)gridDim.x * S::WARPS, gw = (long long)blockIdx.x * S::WARPS + warp;
  const long long i0 = total * gw / nw, i1 = total * (gw + 1) / nw;

  PvCursor ic, cc;
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
    const int sl = kiss % NS;
    if (lane == 0)
      pv5_issue<G>(heads + sl * S::HEAD, pblks + sl * G * R, metab + (ic.npage & 1) * S::META, &full[sl], ic, &tmv, st,
                   cap);
    iv = pv_cursor_next<R>(ic, i1, s, npg_max, 1);
  }

  float acc[NT][8][4];  // [n-tile][16-channel tile][fragment]
  int adj[G][3], base[G];
  bool any_gen = false;
  long long vbytes = 0;
  const uint8_t* vb = nullptr;
  int slot = 0, isl = kiss % NS;
  uint32_t phase = 0;
  for (; cv; slot = slot + 1 == NS ? 0 : slot + 1, phase ^= slot == 0) {
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    // the page meta is double-buffered: page N+2's first stage waits until page N is consumed
    if (iv && (ic.sub != 0 || ic.npage - cc.npage < 2)) {
      if (lane == 0)
        pv5_issue<G>(heads + isl * S::HEAD, pblks + isl * G * R, metab + (ic.npage & 1) * S::META, &full[isl], ic, &tmv,
                     st, cap);
      isl = isl + 1 == NS ? 0 : isl + 1;
      iv = pv_cursor_next<R>(ic, i1, s, npg_max, 1);
    }
    mbar_wait(&full[slot], phase);
    const uint8_t* hd = heads + slot * S::HEAD;
    float* pb = pblks + slot * G * R;
    const uint32_t* md = reinterpret_cast<const uint32_t*>(metab + (cc.npage & 1) * S::META);
    const uint32_t* selm = md;
    const uint32_t* needm = md + G * 8;
    if (cc.sub == 0) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int ti = 0; ti < 8; ++ti) acc[nt][ti][0] = acc[nt][ti][1] = acc[nt][ti][2] = acc[nt][ti][3] = 0.f;
#pragma unroll
      for (int j = 0; j < G; ++j) {
        adj[j][0] = adj[j][1] = adj[j][2] = 0;
        base[j] = 0;
      }
      any_gen = false;
      vbytes = 0;
      vb = s.v_pool + cc.pid * PAGE;
    }
    const int r0 = cc.sub * R;
    const int nvs = min(R, cc.rows - r0);
    const int chk = r0 >> 5;
    const uint32_t vmask = nvs >= 32 ? 0xFFFFFFFFu : ((1u << nvs) - 1u);
    uint32_t um = 0u, wm = 0u, wl = 0u;
#pragma unroll
    for (int j = 0; j < G; ++j) {
      wm |= needm[j * 16 + chk];
      wl |= needm[j * 16 + 8 + chk];
    }
    um = (wm | wl) & vmask;
    vbytes += (long long)nvs * D + (long long)(__popc(wm & vmask) + __popc(wl & vmask)) * (D / 2);
    // rows in the plan: the CUDA-core rule (before p is cleared for them) into gen[]; the two
    // row halves take turns so each (head, channel) entry has one writer at a time
    if (um) {
      if (!any_gen) {
        for (int i = lane; i < G * D; i += 32) gen[i] = 0.f;
        any_gen = true;
      }
      const int half = lane >> 4, cg = lane & 15;
#pragma unroll 1
      for (int i = 0; i < 16; ++i) {
        if (!(((um >> i) | (um >> (16 + i))) & 1u)) continue;  // warp-uniform: row pair (i, 16 + i)
#pragma unroll 1
        for (int hh = 0; hh < 2; ++hh) {
          __syncwarp();
          const int rr = 16 * hh + i;
          if (half == hh && ((um >> rr) & 1u)) {
            const uint2 hv = *reinterpret_cast<const uint2*>(hd + rr * D + (((cg >> 1) ^ (rr & 7)) << 4) + (cg & 1) * 8);
            const Pv5Adj<G> ad = pv5_row_rule<G>(hv, r0 + rr, gen, pb, rr, vb, selm, needm, cc.u, cfg, st.targets);
#pragma unroll
            for (int j = 0; j < G; ++j) {
              adj[j][0] += ad.a[j][0];
              adj[j][1] += ad.a[j][1];
              adj[j][2] += ad.a[j][2];
            }
          }
        }
      }
      __syncwarp();
    }
    // B operand source: p = 0 for selected rows (D6), rows past the length and plan rows
    {
      const bool dead = !((vmask >> lane) & 1u) || ((um >> lane) & 1u);
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const uint32_t sw = selm[j * 8 + chk];
        if (dead || ((sw >> lane) & 1u)) pb[j * R + lane] = 0.f;
        base[j] += nvs - __popc(sw & vmask);
      }
    }
    __syncwarp();
    // two k-steps of 16 tokens
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      uint32_t bf[NT][2];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int n = 8 * nt + g, j = n >> 1;
        if (j < G) {
          const float* pj = pb + j * R + 16 * ks + 2 * t;
          const float x0 = pj[0] * 16384.f, x1 = pj[1] * 16384.f, x8 = pj[8] * 16384.f, x9 = pj[9] * 16384.f;
          const bool lo = n & 1;
          bf[nt][0] = hilo16(x0, lo) | (hilo16(x1, lo) << 16);
          bf[nt][1] = hilo16(x8, lo) | (hilo16(x9, lo) << 16);
        } else {
          bf[nt][0] = bf[nt][1] = 0u;
        }
      }
      const int tok = 16 * ks + (lane & 7) + ((lane >> 3) & 1) * 8;  // the row this lane addresses
#pragma unroll
      for (int tp = 0; tp < 4; ++tp) {  // channel tiles 2tp, 2tp + 1
        const int chunk = 2 * tp + (lane >> 4);
        uint32_t r[4];
        ldsm_x4_trans(r, hd + tok * D + ((chunk ^ (tok & 7)) << 4));
        const uint32_t c80 = 0x80808080u;
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const uint32_t a0 = prmt(r[2 * h2], c80, 0x2404), a1 = prmt(r[2 * h2], c80, 0x3414);
          const uint32_t a2 = prmt(r[2 * h2 + 1], c80, 0x2404), a3 = prmt(r[2 * h2 + 1], c80, 0x3414);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) mma_16816(acc[nt][2 * tp + h2], a0, a1, a2, a3, bf[nt][0], bf[nt][1]);
        }
      }
    }

    if (cc.sub + 1 == cc.nsub) {
      if (lane == 0)
        atomicAdd(reinterpret_cast<unsigned long long*>(st.unit_bytes + (size_t)cc.u * 4 + 1),
                  (unsigned long long)vbytes);
      __syncwarp();
      // lane (g, t): head 4nt + t, channels 16ti + 2g (d0 + d1) and 16ti + 2g + 1 (d2 + d3)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int j = 4 * nt + t;
        if (j < G) {
          const size_t h = (size_t)cc.u * G + j;
          float* dst = st.o_partial + (h * (cap / P) + cc.pg) * D;
#pragma unroll
          for (int ti = 0; ti < 8; ++ti) {
            const int c = 16 * ti + 2 * g;
            float o0 = (acc[nt][ti][0] + acc[nt][ti][1]) * (1.f / 16384.f);
            float o1 = (acc[nt][ti][2] + acc[nt][ti][3]) * (1.f / 16384.f);
            if (any_gen) {
              o0 += gen[j * D + c];
              o1 += gen[j * D + c + 1];
            }
            *reinterpret_cast<float2*>(dst + c) = make_float2(o0, o1);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const int a = warp_sum_i(adj[j][0]), b1 = warp_sum_i(adj[j][1]), c2 = warp_sum_i(adj[j][2]);
        if (lane == 0) {
          unsigned long long* ct = reinterpret_cast<unsigned long long*>(st.counters + ((size_t)cc.u * G + j) * 8 + 3);
          const long long t8 = a + (long long)base[j] * D;
          if (t8) atomicAdd(ct + 0, (unsigned long long)t8);
          if (b1) atomicAdd(ct + 1, (unsigned long long)b1);
          if (c2) atomicAdd(ct + 2, (unsigned long long)c2);
        }
      }
    }
    cv = pv_cursor_next<R>(cc, i1, s, npg_max, 1);
  }
}

// ---------------------------------------------------------------------------
// V head-row tensor map: the pool as rows of 128 B (page p's head rows are rows
// 512p .. 512p+255), box 128 B x 32 rows, 128 B swizzle.  Cached per (pool, size).
// ---------------------------------------------------------------------------
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static bool v_head_tmap(const akv_store_t& s, CUtensorMap* out) {
  static PFN_encodeTiled encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (PFN_encodeTiled) nullptr;
    return (PFN_encodeTiled)fn;
  }();
  if (!encode) return false;
  const long long pages = s.pool_pages > 0 ? s.pool_pages : (long long)s.n_units * s.max_pages;
  struct Entry {
    const void* pool;
    long long pages;
    CUtensorMap map;
  };
  static thread_local Entry cache[8];
  static thread_local int next = 0;
  for (auto& e : cache)
    if (e.pool == s.v_pool && e.pages == pages) {
      *out = e.map;
      return true;
    }
  cuuint64_t dims[2] = {128, (cuuint64_t)pages * 512};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {128, 32};
  cuuint32_t es[2] = {1, 1};
  CUtensorMap m;
  if (encode(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, s.v_pool, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS)
    return false;
  cache[next] = Entry{s.v_pool, pages, m};
  next = (next + 1) % 8;
  *out = m;
  return true;
}

template <int G>
static bool launch_pv5_t(const akv_store_t& s, const akv_cfg_t& cfg, const akv_step_t& st, int max_len,
                         cudaStream_t stream) {
  using S = Pv5Shape<G>;
  CUtensorMap tm;
  if (!v_head_tmap(s, &tm)) return false;
  const int resident = resident_ctas<pv5_kernel<G>>(32 * S::WARPS, S::SMEM);
  const int cap = s.max_pages * P;
  const int npg = (max_len + P - 1) / P;
  const long long items = (long long)s.n_units * npg;
  const int grid = (int)std::min<long long>(resident, std::max<long long>((items + S::WARPS - 1) / S::WARPS, 1));
  launch_pdl(PDL_PV, pv5_kernel<G>, dim3(grid), dim3(32 * S::WARPS), (size_t)S::SMEM, stream, s, cfg, st, cap, npg, tm);
  return true;
}

}  // namespace akv
