// scores_aligned for every (unit, q-head) of a batch.
//
// Prologue (every CTA of a unit, 128 threads = channels): Rule 1
// (rule1_target SPEC.md:157-165, required_mantissa_bits :139-147,
// tier_for_bits :148-156, k_channel_tiers :175-183 with A-K, D1, D2, D8) ->
// per-(head, channel) tier masks and the union fetch bitmaps of the kv-head.
//
// Main loop: one warp per 256-token page; lane = 8 consecutive tokens.  For
// each channel the warp reads one 256 B head-plane row (LDG.64 per lane) and,
// only when the union tier needs them, one 128 B mid row and one 128 B low row
// (predicated LDG.32).  Words are rebuilt with LOP3/PRMT (midpoint fill for
// absent nibbles, HB:160-179) and multiplied into fp32 accumulators with the
// mixed-precision FHFMA (exact fp16 x fp16 products; D9).
// The 1/sqrt(d) scale is applied after accumulation.  Each warp
// also emits its page's (max, sum exp) for the split softmax.
#include "akv_common.cuh"

namespace akv {

// acc += half(a, element E of the pair) * half(qpair, element Q)
template <int E, int Q>
__device__ __forceinline__ float fma_hh(uint32_t a, uint32_t qpair, float c) {
  float d;
  if (E == 0 && Q == 0)
    asm("{\n\t.reg .f16 a0, a1, q0, q1;\n\tmov.b32 {a0, a1}, %1;\n\tmov.b32 {q0, q1}, %2;\n\t"
        "fma.rn.f32.f16 %0, a0, q0, %3;\n\t}"
        : "=f"(d) : "r"(a), "r"(qpair), "f"(c));
  else if (E == 1 && Q == 0)
    asm("{\n\t.reg .f16 a0, a1, q0, q1;\n\tmov.b32 {a0, a1}, %1;\n\tmov.b32 {q0, q1}, %2;\n\t"
        "fma.rn.f32.f16 %0, a1, q0, %3;\n\t}"
        : "=f"(d) : "r"(a), "r"(qpair), "f"(c));
  else if (E == 0 && Q == 1)
    asm("{\n\t.reg .f16 a0, a1, q0, q1;\n\tmov.b32 {a0, a1}, %1;\n\tmov.b32 {q0, q1}, %2;\n\t"
        "fma.rn.f32.f16 %0, a0, q1, %3;\n\t}"
        : "=f"(d) : "r"(a), "r"(qpair), "f"(c));
  else
    asm("{\n\t.reg .f16 a0, a1, q0, q1;\n\tmov.b32 {a0, a1}, %1;\n\tmov.b32 {q0, q1}, %2;\n\t"
        "fma.rn.f32.f16 %0, a1, q1, %3;\n\t}"
        : "=f"(d) : "r"(a), "r"(qpair), "f"(c));
  return d;
}

template <int Q>
__device__ __forceinline__ void fma8(const uint32_t w[4], uint32_t qpair, float acc[8]) {
  acc[0] = fma_hh<0, Q>(w[0], qpair, acc[0]);
  acc[1] = fma_hh<1, Q>(w[0], qpair, acc[1]);
  acc[2] = fma_hh<0, Q>(w[1], qpair, acc[2]);
  acc[3] = fma_hh<1, Q>(w[1], qpair, acc[3]);
  acc[4] = fma_hh<0, Q>(w[2], qpair, acc[4]);
  acc[5] = fma_hh<1, Q>(w[2], qpair, acc[5]);
  acc[6] = fma_hh<0, Q>(w[3], qpair, acc[6]);
  acc[7] = fma_hh<1, Q>(w[3], qpair, acc[7]);
}

struct QkSmem {
  uint4 msk[AKV_MAX_GROUP][D];     // mk, lk, lf, unused
  uint32_t q[AKV_MAX_GROUP][D / 2];  // q pairs, SKIP channels zeroed
  uint32_t fetch[3][4];            // union bitmaps: head / mid / low
  int red[4][AKV_MAX_GROUP];
};

template <int G, bool TRUNC>
__global__ void __launch_bounds__(128) qk_kernel(akv_store_t s, akv_cfg_t cfg, akv_step_t st, int cap,
                                                 float inv_sqrt_d) {
  const int u = blockIdx.y;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = s.lengths[u];
  __shared__ QkSmem sm;

  // ---------------- prologue: Rule 1 tiers per (head, channel) ----------------
  const int c = tid;
  const uint32_t cmw = s.colmax[(size_t)u * D + c] & 0x7FFFu;
  const bool aligned = cfg.force_tier == 0 && !TRUNC;
  int code[G];
  uint32_t qw[G];
  int pe[G];
#pragma unroll
  for (int j = 0; j < G; ++j) {
    qw[j] = st.q[((size_t)u * G + j) * D + c];
    const bool valid = (qw[j] & 0x7FFFu) && cmw && finite16(qw[j]);
    pe[j] = valid ? magexp16(qw[j]) + magexp16(cmw) + 1 : INT_MIN;
    const int m = warp_max_i(pe[j]);
    if (lane == 0) sm.red[warp][j] = m;
  }
  __syncthreads();
  int ucode = 0;
#pragma unroll
  for (int j = 0; j < G; ++j) {
    const int maxpe = max(max(sm.red[0][j], sm.red[1][j]), max(sm.red[2][j], sm.red[3][j]));
    int cd;
    if (!aligned) {
      cd = TRUNC ? 16 : cfg.force_tier;
    } else if (maxpe == INT_MIN) {
      cd = 16;  // degenerate: status reported below, result undefined
    } else {
      const int t = min(max(pe[j] - maxpe + 9 + cfg.margin_bits, 0), 10);  // pe - u - 1 + margin, u = maxpe - 10
      cd = t <= 2 ? 8 : (t <= 6 ? 12 : 16);
      const bool qz = (qw[j] & 0x7FFFu) == 0, cz = cmw == 0;
      if (cfg.zero_skip) {
        if (qz || cz) cd = 0;
      } else {
        if (qz) cd = 8;       // D1
        else if (cz) cd = 16; // D2
      }
    }
    code[j] = cd;
    ucode = max(ucode, cd);
    const TierMask tm = tier_mask(cd);
    sm.msk[j][c] = make_uint4(tm.mk, tm.lk, tm.lf, 0u);
    const uint32_t qe = cd ? qw[j] : 0u;
    const uint32_t qo = __shfl_down_sync(0xFFFFFFFFu, qe, 1);
    if ((c & 1) == 0) sm.q[j][c >> 1] = qe | (qo << 16);
  }
  {
    const uint32_t bh = __ballot_sync(0xFFFFFFFFu, ucode >= 8);
    const uint32_t bm = __ballot_sync(0xFFFFFFFFu, ucode >= 12);
    const uint32_t bl = __ballot_sync(0xFFFFFFFFu, ucode >= 16);
    if (lane == 0) {
      sm.fetch[0][warp] = bh;
      sm.fetch[1][warp] = bm;
      sm.fetch[2][warp] = bl;
    }
  }
  if (blockIdx.x == 0) {  // per-step bookkeeping, once per unit
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const size_t h = (size_t)u * G + j;
      st.k_tiers[h * D + c] = (uint8_t)code[j];
      const int n8 = __syncthreads_count(code[j] == 8);
      const int n12 = __syncthreads_count(code[j] == 12);
      const int n16 = __syncthreads_count(code[j] == 16);
      const int badq = __syncthreads_count(!finite16(qw[j]));
      if (tid == 0) {
        int64_t* ct = st.counters + h * 8;
        ct[0] = (int64_t)n8 * n;
        ct[1] = (int64_t)n12 * n;
        ct[2] = (int64_t)n16 * n;
        ct[3] = ct[4] = ct[5] = ct[6] = ct[7] = 0;
        const int maxpe = max(max(sm.red[0][j], sm.red[1][j]), max(sm.red[2][j], sm.red[3][j]));
        long long stw = 0;
        if (badq) stw = status_word(AKV_STATUS_BAD_Q, 0);
        else if (aligned && maxpe == INT_MIN) stw = status_word(AKV_STATUS_DEGENERATE, 0);
        st.status[h] = stw;
      }
    }
    const int uh = __syncthreads_count(ucode >= 8);
    const int um = __syncthreads_count(ucode >= 12);
    const int ul = __syncthreads_count(ucode >= 16);
    if (tid == 0) {
      st.unit_bytes[(size_t)u * 4 + 0] = (int64_t)n * uh + (int64_t)(n / 2) * (um + ul);
      st.unit_bytes[(size_t)u * 4 + 1] = 0;
    }
  }
  __syncthreads();

  // ---------------- main loop: one page per warp ----------------
  const int pg = blockIdx.x * 4 + warp;
  if (pg * P >= n) return;
  const uint8_t* base = page_ptr(s.k_pool, s.page_table, s.max_pages, u, pg);
  const int tok0 = pg * P + lane * 8;
  const bool lv = tok0 < n;
  const uint8_t* hp = base + lane * 8;
  const uint8_t* mp = base + MID + lane * 4;
  const uint8_t* lp = base + LOW + lane * 4;
  const uint64_t pol = evict_first_policy();

  uint32_t tkm = 0xFFFFFFFFu, tf = 0u;
  if (TRUNC) {
    const int kb = cfg.trunc_bits - 6;
    const uint32_t km = (0xFFFFu << (10 - kb)) & 0xFFFFu;
    const uint32_t fill = kb < 10 ? (1u << (9 - kb)) : 0u;
    tkm = km | (km << 16);
    tf = fill | (fill << 16);
  }

  float acc[G][8];
#pragma unroll
  for (int j = 0; j < G; ++j)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[j][e] = 0.f;

#pragma unroll 1
  for (int wd = 0; wd < 4; ++wd) {
    const uint32_t fh = lv ? sm.fetch[0][wd] : 0u;
    const uint32_t fm = lv ? sm.fetch[1][wd] : 0u;
    const uint32_t fl = lv ? sm.fetch[2][wd] : 0u;
#pragma unroll
    for (int cb = 0; cb < 32; cb += 8) {
      uint2 hv[8];
      uint32_t mv[8], lvv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int ch = wd * 32 + cb + i;
        const uint32_t bit = 1u << (cb + i);
        hv[i] = make_uint2(0u, 0u);
        mv[i] = 0u;
        lvv[i] = 0u;
        if (fh & bit) hv[i] = ld_stream_u64(hp + ch * P, pol);
        if (fm & bit) mv[i] = ld_stream_u32(mp + ch * (P / 2), pol);
        if (fl & bit) lvv[i] = ld_stream_u32(lp + ch * (P / 2), pol);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int ch = wd * 32 + cb + i;
#pragma unroll
        for (int j = 0; j < G; ++j) {
          const uint4 mk = sm.msk[j][ch];
          uint32_t w[4];
          assemble8(hv[i].x, hv[i].y, bsel(mk.x, mv[i], 0x88888888u), bsel(mk.y, lvv[i], mk.z), w);
          if (TRUNC) {
#pragma unroll
            for (int k = 0; k < 4; ++k) w[k] = (w[k] & tkm) | tf;
          }
          const uint32_t qp = sm.q[j][ch >> 1];
          if (i & 1)
            fma8<1>(w, qp, acc[j]);
          else
            fma8<0>(w, qp, acc[j]);
        }
      }
    }
  }

  // ---------------- epilogue: scores + page softmax stats ----------------
  const int nv = min(max(n - tok0, 0), 8);
#pragma unroll
  for (int j = 0; j < G; ++j) {
    const size_t h = (size_t)u * G + j;
    float sv[8];
    float m = -INFINITY;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      sv[e] = acc[j][e] * inv_sqrt_d;
      if (e < nv) m = fmaxf(m, sv[e]);
    }
    m = warp_max(m);
    float l = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (e < nv) l += expf(sv[e] - m);
    l = warp_sum(l);
    float* out = st.scores + h * cap + tok0;
    if (nv == 8) {
      reinterpret_cast<float4*>(out)[0] = make_float4(sv[0], sv[1], sv[2], sv[3]);
      reinterpret_cast<float4*>(out)[1] = make_float4(sv[4], sv[5], sv[6], sv[7]);
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (e < nv) out[e] = sv[e];
    }
    if (lane == 0) {
      float* ps = st.page_stats + (h * s.max_pages + pg) * 2;
      ps[0] = m;
      ps[1] = l;
    }
  }
}

template <int G>
static void launch_qk_g(const akv_store_t& s, const akv_cfg_t& cfg, const akv_step_t& st, int max_len,
                        cudaStream_t stream) {
  const int cap = s.max_pages * P;
  const int npg = (max_len + P - 1) / P;
  dim3 grid((max(npg, 1) + 3) / 4, s.n_units);
  const float isd = (float)(1.0 / 11.313708498984761);  // 1/sqrt(128)
  if (cfg.trunc_bits)
    qk_kernel<G, true><<<grid, 128, 0, stream>>>(s, cfg, st, cap, isd);
  else
    qk_kernel<G, false><<<grid, 128, 0, stream>>>(s, cfg, st, cap, isd);
}

void launch_qk(const akv_store_t& s, const akv_cfg_t& cfg, const akv_step_t& st, int max_len, cudaStream_t stream) {
  switch (cfg.group) {
    case 1: launch_qk_g<1>(s, cfg, st, max_len, stream); break;
    case 2: launch_qk_g<2>(s, cfg, st, max_len, stream); break;
    case 4: launch_qk_g<4>(s, cfg, st, max_len, stream); break;
    case 8: launch_qk_g<8>(s, cfg, st, max_len, stream); break;
  }
}

}  // namespace akv
