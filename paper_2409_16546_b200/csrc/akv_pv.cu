// output_aligned for every (unit, q-head), split-K over
// pages: one warp per 256-token V page, CTA = 4 pages, partial o per CTA.
//
// Per row t and head j the warp first decides a mode (prologue, one lane per
// row):  SKIP (t selected during estimation, D6: its T16 contribution is
// already in o_est), a uniform tier (T8 when p_t = 0 (D5) or when the RowMax
// superset bound proves every element of the row needs <= 2 kept bits (H6);
// forced tiers; the row strategy D7), or ELEMENT (per-element rule from the
// head byte's exponent, D4).  The union over the kv-head's q-heads decides
// which 64 B nibble rows are fetched; per-element truncation is then applied
// exactly, so the masks match the oracle bit-for-bit.
//
// Lane mapping: 16 lanes per row, 8 channels per lane (LDG.64 head + LDG.32
// mid/low); two rows per warp instruction.  fp16 -> fp32 via HADD2.F32 and the
// packed FFMA2 accumulate p_t * V~[t, r] in fp32 (>= 24-bit).
#include "akv_common.cuh"

namespace akv {

enum : uint8_t { M_SKIP = 0, M_ELEM = 1, M_T8 = 8, M_T12 = 12, M_T16 = 16 };

template <int G>
struct PvLayout {
  static constexpr size_t p_off = 0;                                  // float [4][G][P]
  static constexpr size_t ep_off = p_off + sizeof(float) * 4 * G * P;  // int16 [4][G][P]
  static constexpr size_t mode_off = ep_off + sizeof(int16_t) * 4 * G * P;  // u8 [4][G][P]
  static constexpr size_t fl_off = mode_off + 4 * G * P;              // u8 [4][P]
  static constexpr size_t g_off = fl_off + 4 * P;                     // int [G][D]
  static constexpr size_t bytes = g_off + sizeof(int) * G * D;
};

template <int G, bool TRUNC, bool EXPORT>
__global__ void __launch_bounds__(128) pv_kernel(akv_store_t s, akv_cfg_t cfg, akv_step_t st, int cap, int nblk) {
  using L = PvLayout<G>;
  extern __shared__ __align__(16) uint8_t smem[];
  float* s_p = reinterpret_cast<float*>(smem + L::p_off);
  int16_t* s_ep = reinterpret_cast<int16_t*>(smem + L::ep_off);
  uint8_t* s_mode = smem + L::mode_off;
  uint8_t* s_fl = smem + L::fl_off;
  int* s_g = reinterpret_cast<int*>(smem + L::g_off);
  __shared__ long long s_cnt[4][G][3];

  const int u = blockIdx.y;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = s.lengths[u];
  if (blockIdx.x * 4 * P >= n) return;  // whole CTA beyond this unit (uniform)
  const int pg = blockIdx.x * 4 + warp;
  const bool wv = pg * P < n;
  const bool aligned = cfg.force_tier == 0 && !TRUNC;
  const int uniform = TRUNC ? 16 : cfg.force_tier;

  // per-head element thresholds: keep mid <=> max(bexp,1) + e_p > g_r (g_r = 17 + target_r - margin)
#pragma unroll
  for (int j = 0; j < G; ++j) {
    const int tg = st.targets[((size_t)u * G + j) * D + tid];
    s_g[j * D + tid] = tg == AKV_TARGET_UNKNOWN ? -(1 << 20) : 17 + tg - cfg.margin_bits;
  }

  // ---------------- prologue: row modes (one lane per row) ----------------
  long long vbytes = 0;
  if (wv) {
    int min_t[G], unk[G];
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const int32_t* hm = st.head_meta + ((size_t)u * G + j) * 4;
      min_t[j] = hm[1];
      unk[j] = hm[2];
    }
    for (int r = lane; r < P; r += 32) {
      const int t = pg * P + r;
      uint8_t fl = 0;
      if (t < n) {
        const uint32_t rm = s.rowmax[(size_t)u * s.max_pages * P + t];
        const int e_rm = max(bexp16(rm), 1) - 15;  // D4 bound on every element's e_v
#pragma unroll
        for (int j = 0; j < G; ++j) {
          const size_t h = (size_t)u * G + j;
          uint8_t mode;
          float p = 0.f;
          int ep = -30000;
          if (!aligned) {
            mode = (uint8_t)uniform;
            p = st.probs[h * cap + t];
          } else {
            const bool sel = (st.sel_bits[h * (cap >> 5) + (t >> 5)] >> (t & 31)) & 1u;
            p = st.probs[h * cap + t];
            if (p > 0.f) ep = floor_log2f(p);
            if (sel) {
              mode = M_SKIP;
              p = 0.f;
            } else if (cfg.strategy == 1) {  // row strategy (D7)
              if (unk[j]) mode = M_T16;
              else if (p == 0.f || rm == 0) mode = M_T8;
              else {
                const int tr = min(max(ep + magexp16(rm) + 1 - min_t[j] - 1 + cfg.margin_bits, 0), 10);
                mode = tr <= 2 ? M_T8 : (tr <= 6 ? M_T12 : M_T16);
              }
            } else if (p == 0.f) {
              mode = M_T8;  // D5
            } else if (unk[j]) {
              mode = M_ELEM;
              fl |= 6;
            } else {
              const int bound = ep + e_rm + 1 - min_t[j] - 1 + cfg.margin_bits;  // superset t_req (H6)
              if (bound > 2) {
                mode = M_ELEM;
                fl |= 2;
                if (bound > 6) fl |= 4;
              } else {
                mode = M_T8;
              }
            }
          }
          if (mode != M_SKIP) fl |= 1;
          if (mode == M_T12) fl |= 2;
          if (mode == M_T16) fl |= 6;
          s_p[(warp * G + j) * P + r] = p;
          s_ep[(warp * G + j) * P + r] = (int16_t)ep;
          s_mode[(warp * G + j) * P + r] = mode;
        }
      } else {
#pragma unroll
        for (int j = 0; j < G; ++j) s_mode[(warp * G + j) * P + r] = M_SKIP;
      }
      s_fl[warp * P + r] = fl;
      vbytes += (fl & 1 ? D : 0) + (fl & 2 ? D / 2 : 0) + (fl & 4 ? D / 2 : 0);
    }
  }
  __syncthreads();

  // ---------------- main loop ----------------
  const int half = lane >> 4, cl = lane & 15;
  float2 acc[G][4];
  long long c8[G], c12[G], c16[G];
#pragma unroll
  for (int j = 0; j < G; ++j) {
    c8[j] = c12[j] = c16[j] = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[j][k] = make_float2(0.f, 0.f);
  }
  uint32_t tkm = 0xFFFFFFFFu, tf = 0u;
  if (TRUNC) {
    const int kb = cfg.trunc_bits - 6;
    const uint32_t km = (0xFFFFu << (10 - kb)) & 0xFFFFu;
    const uint32_t fill = kb < 10 ? (1u << (9 - kb)) : 0u;
    tkm = km | (km << 16);
    tf = fill | (fill << 16);
  }

  if (wv) {
    const uint8_t* base = page_ptr(s.v_pool, s.page_table, s.max_pages, u, pg);
    const uint8_t* hp = base + cl * 8;
    const uint8_t* mp = base + MID + cl * 4;
    const uint8_t* lp = base + LOW + cl * 4;
    const uint64_t pol = evict_first_policy();
    const uint8_t* flp = s_fl + warp * P;
    const int rows_valid = min(n - pg * P, P);
#pragma unroll 1
    for (int rb = 0; rb < P; rb += 16) {
      if (rb >= rows_valid) break;
      uint2 hv[8];
      uint32_t mv[8], lw[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = rb + 2 * i + half;
        const uint8_t f = flp[r];
        hv[i] = make_uint2(0u, 0u);
        mv[i] = 0u;
        lw[i] = 0u;
        if (f & 1) hv[i] = ld_stream_u64(hp + r * D, pol);
        if (f & 2) mv[i] = ld_stream_u32(mp + r * (D / 2), pol);
        if (f & 4) lw[i] = ld_stream_u32(lp + r * (D / 2), pol);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = rb + 2 * i + half;
#pragma unroll
        for (int j = 0; j < G; ++j) {
          const int idx = (warp * G + j) * P + r;
          const uint8_t mode = s_mode[idx];
          if (mode == M_SKIP) {
            if (EXPORT && st.v_tiers && r < rows_valid) {  // selected row: read at T16 by the estimate (D6)
              uint8_t* dst = st.v_tiers + (((size_t)u * G + j) * cap + pg * P + r) * D + cl * 8;
              *reinterpret_cast<uint2*>(dst) = make_uint2(0x10101010u, 0x10101010u);
            }
            continue;
          }
          const float p = s_p[idx];
          uint32_t w[4];
          uint32_t codes_lo = 0, codes_hi = 0;  // export: 8 codes packed as bytes
          if (mode != M_ELEM) {
            const TierMask tm = tier_mask(mode);
            assemble8(hv[i].x, hv[i].y, bsel(tm.mk, mv[i], 0x88888888u), bsel(tm.lk, lw[i], tm.lf), w);
            if (mode == M_T8) c8[j] += 8;
            else if (mode == M_T12) c12[j] += 8;
            else c16[j] += 8;
            if (EXPORT) codes_lo = codes_hi = (uint32_t)mode * 0x01010101u;
          } else {
            assemble8(hv[i].x, hv[i].y, mv[i], lw[i], w);
            const int ep = s_ep[idx];
            const int4 g0 = *reinterpret_cast<const int4*>(s_g + j * D + cl * 8);
            const int4 g1 = *reinterpret_cast<const int4*>(s_g + j * D + cl * 8 + 4);
            const int gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const uint32_t hb = ((e < 4 ? hv[i].x : hv[i].y) >> (8 * (e & 3))) & 0xFFu;
              const int E = max((int)((hb >> 2) & 31u), 1) + ep;
              const bool km = E > gg[e], kl = E > gg[e] + 4;
              const int sh = 16 * (e & 1);
              uint32_t w16 = (w[e >> 1] >> sh) & 0xFFFFu;
              w16 = kl ? w16 : (km ? ((w16 & 0xFFF0u) | 0x8u) : ((w16 & 0xFF00u) | 0x80u));
              w[e >> 1] = (w[e >> 1] & ~(0xFFFFu << sh)) | (w16 << sh);
              const uint32_t cd = kl ? 16u : (km ? 12u : 8u);
              if (kl) c16[j] += 1;
              else if (km) c12[j] += 1;
              else c8[j] += 1;
              if (EXPORT) {
                if (e < 4) codes_lo |= cd << (8 * e);
                else codes_hi |= cd << (8 * (e - 4));
              }
            }
          }
          if (TRUNC) {
#pragma unroll
            for (int k = 0; k < 4; ++k) w[k] = (w[k] & tkm) | tf;
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) acc[j][k] = ffma2_scalar(half2_bits_to_float2(w[k]), p, acc[j][k]);
          if (EXPORT && st.v_tiers) {
            const size_t h = (size_t)u * G + j;
            uint8_t* dst = st.v_tiers + (h * cap + pg * P + r) * D + cl * 8;
            *reinterpret_cast<uint2*>(dst) = make_uint2(codes_lo, codes_hi);
          }
        }
      }
    }
  }

  // ---------------- epilogue: reduce partial o, counters ----------------
  __syncthreads();  // smem p/ep/mode no longer needed: reuse as reduction buffer
  float* red = reinterpret_cast<float*>(smem);  // [4][G][D]
#pragma unroll
  for (int j = 0; j < G; ++j) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      acc[j][k].x += __shfl_xor_sync(0xFFFFFFFFu, acc[j][k].x, 16);
      acc[j][k].y += __shfl_xor_sync(0xFFFFFFFFu, acc[j][k].y, 16);
    }
    if (half == 0) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        red[(warp * G + j) * D + cl * 8 + 2 * k] = acc[j][k].x;
        red[(warp * G + j) * D + cl * 8 + 2 * k + 1] = acc[j][k].y;
      }
    }
    const long long a = warp_sum_ll(c8[j]), b = warp_sum_ll(c12[j]), c = warp_sum_ll(c16[j]);
    if (lane == 0) {
      s_cnt[warp][j][0] = a;
      s_cnt[warp][j][1] = b;
      s_cnt[warp][j][2] = c;
    }
  }
  vbytes = warp_sum_ll(vbytes);
  __syncthreads();
#pragma unroll
  for (int j = 0; j < G; ++j) {
    const size_t h = (size_t)u * G + j;
    const float v = red[(0 * G + j) * D + tid] + red[(1 * G + j) * D + tid] + red[(2 * G + j) * D + tid] +
                    red[(3 * G + j) * D + tid];
    st.o_partial[(h * nblk + blockIdx.x) * D + tid] = v;
    if (tid < 3) {
      const long long tot = s_cnt[0][j][tid] + s_cnt[1][j][tid] + s_cnt[2][j][tid] + s_cnt[3][j][tid];
      atomicAdd(reinterpret_cast<unsigned long long*>(st.counters + h * 8 + 3 + tid), (unsigned long long)tot);
    }
  }
  if (lane == 0 && vbytes)
    atomicAdd(reinterpret_cast<unsigned long long*>(st.unit_bytes + (size_t)u * 4 + 1), (unsigned long long)vbytes);
}

// o = o_est + sum of the unit's partials, fixed order (deterministic).
__global__ void __launch_bounds__(128) combine_kernel(akv_store_t s, akv_cfg_t cfg, akv_step_t st, int nblk) {
  const int h = blockIdx.x;
  const int u = h / cfg.group;
  const int n = s.lengths[u];
  const int nb = (n + 4 * P - 1) / (4 * P);
  float acc = st.o_est[(size_t)h * D + threadIdx.x];
  for (int b = 0; b < nb; ++b) acc += st.o_partial[((size_t)h * nblk + b) * D + threadIdx.x];
  st.o[(size_t)h * D + threadIdx.x] = acc;
}

template <int G, bool TRUNC, bool EXPORT>
static void launch_pv_t(const akv_store_t& s, const akv_cfg_t& cfg, const akv_step_t& st, int max_len,
                        cudaStream_t stream) {
  const int cap = s.max_pages * P;
  const int nblk = (s.max_pages + 3) / 4;
  const int npg = (max_len + P - 1) / P;
  dim3 grid((max(npg, 1) + 3) / 4, s.n_units);
  const size_t bytes = PvLayout<G>::bytes;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(pv_kernel<G, TRUNC, EXPORT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    attr_set = true;
  }
  pv_kernel<G, TRUNC, EXPORT><<<grid, 128, bytes, stream>>>(s, cfg, st, cap, nblk);
}

template <int G>
static void launch_pv_g(const akv_store_t& s, const akv_cfg_t& cfg, const akv_step_t& st, int max_len,
                        cudaStream_t stream) {
  const bool ex = st.v_tiers != nullptr;
  if (cfg.trunc_bits) {
    if (ex) launch_pv_t<G, true, true>(s, cfg, st, max_len, stream);
    else launch_pv_t<G, true, false>(s, cfg, st, max_len, stream);
  } else {
    if (ex) launch_pv_t<G, false, true>(s, cfg, st, max_len, stream);
    else launch_pv_t<G, false, false>(s, cfg, st, max_len, stream);
  }
}

void launch_pv(const akv_store_t& s, const akv_cfg_t& cfg, const akv_step_t& st, int max_len, cudaStream_t stream) {
  switch (cfg.group) {
    case 1: launch_pv_g<1>(s, cfg, st, max_len, stream); break;
    case 2: launch_pv_g<2>(s, cfg, st, max_len, stream); break;
    case 4: launch_pv_g<4>(s, cfg, st, max_len, stream); break;
    case 8: launch_pv_g<8>(s, cfg, st, max_len, stream); break;
  }
}

void launch_combine(const akv_store_t& s, const akv_cfg_t& cfg, const akv_step_t& st, cudaStream_t stream) {
  const int nblk = (s.max_pages + 3) / 4;
  combine_kernel<<<s.n_units * cfg.group, D, 0, stream>>>(s, cfg, st, nblk);
}

}  // namespace akv
