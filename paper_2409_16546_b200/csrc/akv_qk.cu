// scores_aligned for every (unit, q-head) of a batch.
// Two kernels: qk_kernel below (G = 1, 2) and qk5_kernel (GQA groups G = 4, 8,
// tensor cores; further down).
//
// Direct-load streaming kernel: every warp owns a contiguous range of
// (unit, page) items (balanced split over all resident warps; no shared-memory
// staging, no cross-warp synchronisation).  Per item the warp
//
//  1. (once per unit) evaluates Rule 1 for the unit's q-heads
//     (rule1_target SPEC.md:157-165, required_mantissa_bits :139-147,
//     tier_for_bits :148-156, k_channel_tiers :175-183, SURVEY App. A
//     A-K/D1/D2/D8) and builds its channel list in shared memory ordered by
//     union class: T8 channels first (head plane only), then T12/T16
//     channels; SKIP channels are dropped (0 bits read).  The warp that owns
//     a unit's page 0 writes the per-step bookkeeping (K tiers, K counters,
//     status, plane bytes);
//  2. streams the page, half-warp per channel row, lane = 16 consecutive
//     tokens: one LDG.128 covers two listed channels' 256 B head-plane rows;
//     only T12/T16 channels add an LDG.64 of their 128 B mid row (+ the low
//     row for T16).  The lists are padded per class to 8 channels so every
//     batch is homogeneous (no per-channel branches).  Loads run two batches
//     of 8 channels ahead of the math, straight into registers (L1
//     no-allocate, L2 evict-first);
//  3. rebuilds fp16 words with PRMT/LOP3 (midpoint fill for absent nibbles,
//     HB:160-179) and accumulates q_c * K~ with the mixed-precision FHFMA
//     (exact fp16 x fp16 products, fp32 sums, D9);
//  4. scales by 1/sqrt(d) after accumulation and writes the
//     page's scores plus a (max, sum exp) pair per 32-token chunk for the
//     split softmax.
// Each page's result is independent of which warp computes it: deterministic.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "akv_common.cuh"

namespace akv {

constexpr int QK_WARPS = 4;  // warps per CTA

template <int G>
struct QkShape {
  // resident CTAs per SM (register budget: 64K / (128 threads * MINB))
  static constexpr int HG = G < 4 ? G : 4;          // q-heads per pass over a page (accumulator budget)
  static constexpr int MINB = G == 1 ? 3 : 2;
};

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

// Per-warp unit state in shared memory.  List positions: T8 class in
// [0, n8p), T12/T16 class in [n8p, nlist), each padded to a multiple of 8 with
// copies of the class's first channel (q = 0: adds nothing, row already in
// flight).  Batch b = positions 8b..8b+7; lane (half h, i) handles position
// 8b + 2i + h.  Per-lane arrays are stored at slot 8b + 4h + i so one LDS.128
// fetches a lane's four values of a batch.
template <int G>
struct alignas(16) QkWarp {
  uint32_t off[D + 16];                 // slot -> channel * P
  uint32_t qrep[G][D + 16];             // slot -> q | q << 16 (fp16), 0 for SKIP heads / pads
  uint2 hm[G > 1 ? G : 1][D + 16];      // slot -> per-head (keep, fill) word masks (T12/T16 class, G > 1)
  uint32_t low[(D + 16) / 32 + 1];      // slot bitmask: T16 (low row needed)
  int n8p, nlist, unit, pad;
};

__device__ __forceinline__ int qk_slot(int pos) { return (pos & ~7) | ((pos & 1) << 2) | ((pos >> 1) & 3); }

struct KBatch {
  uint4 h[4];
  uint2 m[4], l[4];
};

template <int G>
__device__ __forceinline__ void k_load(KBatch& X, const QkWarp<G>& ws, int b, bool full, const uint8_t* base,
                                       int l16, int half, uint64_t pol) {
  const uint4 o = *reinterpret_cast<const uint4*>(&ws.off[8 * b + 4 * half]);
  const uint32_t ov[4] = {o.x, o.y, o.z, o.w};
  const uint32_t lowm = (ws.low[(8 * b) >> 5] >> ((8 * b + 4 * half) & 31)) & 0xFu;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    X.h[i] = ld_stream_u128(base + ov[i] + l16 * 16, pol);
    if (full) {
      const uint8_t* mrow = base + MID + (ov[i] >> 1) + l16 * 8;
      X.m[i] = ld_stream_u64(mrow, pol);
      X.l[i] = make_uint2(0x88888888u, 0x88888888u);
      if ((lowm >> i) & 1u) X.l[i] = ld_stream_u64(mrow + (LOW - MID), pol);
    } else if (G > 1) {
      // T8 words through the full rebuild: mid nibble 8, low nibble 0 = the 0x80 midpoint fill
      X.m[i] = make_uint2(0x88888888u, 0x88888888u);
      X.l[i] = make_uint2(0u, 0u);
    }
  }
}

template <int HG, bool FULL, bool TRUNC, int G>
__device__ __forceinline__ void k_compute(const KBatch& X, const QkWarp<G>& ws, int b, int half, int j0,
                                          float (&acc)[HG][16], uint32_t tkm, uint32_t tf) {
  const int sl = 8 * b + 4 * half;
  uint32_t qv[HG][4];
#pragma unroll
  for (int jj = 0; jj < HG; ++jj) {
    const uint4 q = *reinterpret_cast<const uint4*>(&ws.qrep[j0 + jj][sl]);
    qv[jj][0] = q.x;
    qv[jj][1] = q.y;
    qv[jj][2] = q.z;
    qv[jj][3] = q.w;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint32_t w[8];  // 16 tokens as half2 words
    if (FULL) {
      assemble8(X.h[i].x, X.h[i].y, X.m[i].x, X.l[i].x, w);
      assemble8(X.h[i].z, X.h[i].w, X.m[i].y, X.l[i].y, w + 4);
    } else {
      const uint32_t c80 = 0x80808080u;
      const uint32_t hv[4] = {X.h[i].x, X.h[i].y, X.h[i].z, X.h[i].w};
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        w[2 * r] = prmt(hv[r], c80, 0x1404);
        w[2 * r + 1] = prmt(hv[r], c80, 0x3424);
      }
    }
    if (TRUNC) {
#pragma unroll
      for (int k = 0; k < 8; ++k) w[k] = (w[k] & tkm) | tf;
    }
#pragma unroll
    for (int jj = 0; jj < HG; ++jj) {
      uint32_t wj[8];
      if (G > 1 && FULL) {
        const uint2 hm = ws.hm[j0 + jj][sl + i];
#pragma unroll
        for (int k = 0; k < 8; ++k) wj[k] = (w[k] & hm.x) | hm.y;
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) wj[k] = w[k];
      }
      fma8<0>(wj, qv[jj][i], acc[jj]);
      fma8<0>(wj + 4, qv[jj][i], acc[jj] + 8);
    }
  }
}

// Rule 1 for unit u, all G heads: per-head channel codes (0 SKIP, 8, 12, 16),
// their union over the group, and (book) the per-step bookkeeping.
// Lane l owns channels l + 32k (k = 0..3).
template <int G, bool TRUNC>
__device__ __forceinline__ void k_rule1(const akv_store_t& s, const akv_cfg_t& cfg, const akv_step_t& st, int u,
                                        int n, bool book, uint32_t (&qw)[G][4], int (&code)[G][4],
                                        int (&ucode)[4]) {
  const int lane = threadIdx.x & 31;
  const bool aligned = cfg.force_tier == 0 && !TRUNC;
  uint32_t cm[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) ucode[k] = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) cm[k] = s.colmax[(size_t)u * D + lane + 32 * k] & 0x7FFFu;
#pragma unroll
  for (int j = 0; j < G; ++j)
#pragma unroll
    for (int k = 0; k < 4; ++k) qw[j][k] = st.q[((size_t)u * G + j) * D + lane + 32 * k];
#pragma unroll
  for (int j = 0; j < G; ++j) {
    int pe[4], mx = INT_MIN;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool valid = (qw[j][k] & 0x7FFFu) && cm[k] && finite16(qw[j][k]);
      pe[k] = valid ? magexp16(qw[j][k]) + magexp16(cm[k]) + 1 : INT_MIN;
      mx = max(mx, pe[k]);
    }
    const int maxpe = warp_max_i(mx);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int cd;
      if (!aligned) {
        cd = TRUNC ? 16 : cfg.force_tier;
      } else if (maxpe == INT_MIN) {
        cd = 16;  // degenerate: status reported below, output undefined
      } else {
        const int t = min(max(pe[k] - maxpe + 9 + cfg.margin_bits, 0), 10);  // pe - u - 1 + margin, u = maxpe - 10
        cd = t <= 2 ? 8 : (t <= 6 ? 12 : 16);
        const bool qz = (qw[j][k] & 0x7FFFu) == 0, cz = cm[k] == 0;
        if (cfg.zero_skip) {
          if (qz || cz) cd = 0;
        } else if (qz) {
          cd = 8;  // D1
        } else if (cz) {
          cd = 16;  // D2
        }
      }
      code[j][k] = cd;
      ucode[k] = max(ucode[k], cd);
    }
    if (book) {  // per-step bookkeeping, once per unit (the page-0 item)
      const size_t h = (size_t)u * G + j;
      int c8 = 0, c12 = 0, c16 = 0, bad = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        st.k_tiers[h * D + lane + 32 * k] = (uint8_t)code[j][k];
        c8 += __popc(__ballot_sync(0xFFFFFFFFu, code[j][k] == 8));
        c12 += __popc(__ballot_sync(0xFFFFFFFFu, code[j][k] == 12));
        c16 += __popc(__ballot_sync(0xFFFFFFFFu, code[j][k] == 16));
        bad += __popc(__ballot_sync(0xFFFFFFFFu, !finite16(qw[j][k])));
      }
      if (lane == 0) {
        int64_t* ct = st.counters + h * 8;
        ct[0] = (int64_t)c8 * n;
        ct[1] = (int64_t)c12 * n;
        ct[2] = (int64_t)c16 * n;
        ct[3] = ct[4] = ct[5] = ct[6] = ct[7] = 0;
        long long w = 0;
        if (bad) w = status_word(AKV_STATUS_BAD_Q, 0);
        else if (aligned && maxpe == INT_MIN) w = status_word(AKV_STATUS_DEGENERATE, 0);
        st.status[h] = w;
      }
    }
  }
  if (book) {
    int n8 = 0, nf = 0, n16 = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      n8 += __popc(__ballot_sync(0xFFFFFFFFu, ucode[k] == 8));
      nf += __popc(__ballot_sync(0xFFFFFFFFu, ucode[k] >= 12));
      n16 += __popc(__ballot_sync(0xFFFFFFFFu, ucode[k] == 16));
    }
    if (lane == 0) {
      st.unit_bytes[(size_t)u * 4 + 0] = (int64_t)n * (n8 + nf) + (int64_t)(n / 2) * (nf + n16);
      st.unit_bytes[(size_t)u * 4 + 1] = 0;
    }
  }
}

// Rule 1 + the warp's channel lists for the direct-load kernels.
template <int G, bool TRUNC>
__device__ void k_prologue(QkWarp<G>& ws, const akv_store_t& s, const akv_cfg_t& cfg, const akv_step_t& st, int u,
                           int n, bool book) {
  const int lane = threadIdx.x & 31;
  uint32_t qw[G][4];
  int code[G][4], ucode[4];
  k_rule1<G, TRUNC>(s, cfg, st, u, n, book, qw, code, ucode);
  // lists: T8 class first, then T12/T16 (ascending channel inside each class)
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t b8[4], bf[4];
  int n8 = 0, nf = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    b8[k] = __ballot_sync(0xFFFFFFFFu, ucode[k] == 8);
    bf[k] = __ballot_sync(0xFFFFFFFFu, ucode[k] >= 12);
    n8 += __popc(b8[k]);
    nf += __popc(bf[k]);
  }
  const int n8p = (n8 + 7) & ~7, nlp = n8p + ((nf + 7) & ~7);
  for (int i = lane; i < (D + 16) / 32 + 1; i += 32) ws.low[i] = 0u;
  __syncwarp();
  int base8 = 0, basef = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int c = lane + 32 * k;
    int pos = -1;
    if (ucode[k] == 8) pos = base8 + __popc(b8[k] & lt);
    else if (ucode[k] >= 12) pos = n8p + basef + __popc(bf[k] & lt);
    if (pos >= 0) {
      const int sl = qk_slot(pos);
      ws.off[sl] = (uint32_t)c * P;
      if (ucode[k] == 16) atomicOr(&ws.low[sl >> 5], 1u << (sl & 31));
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const uint32_t qh = code[j][k] ? (qw[j][k] & 0xFFFFu) : 0u;
        ws.qrep[j][sl] = qh | (qh << 16);
        if (G > 1) {
          const int cd = code[j][k];
          ws.hm[j][sl] = cd >= 16 ? make_uint2(0xFFFFFFFFu, 0u)
                                  : (cd == 12 ? make_uint2(0xFFF0FFF0u, 0x00080008u) : make_uint2(0xFF00FF00u, 0x00800080u));
        }
      }
    }
    base8 += __popc(b8[k]);
    basef += __popc(bf[k]);
  }
  __syncwarp();
  // pads: copies of the class's first channel (row already in flight) with q = 0
  const uint32_t off8 = n8 ? ws.off[qk_slot(0)] : 0u, offf = nf ? ws.off[qk_slot(n8p)] : 0u;
  const bool low_f = nf ? ((ws.low[qk_slot(n8p) >> 5] >> (qk_slot(n8p) & 31)) & 1u) : false;
  __syncwarp();
  for (int pos = lane; pos < nlp; pos += 32) {
    const bool pad = pos < n8p ? pos >= n8 : pos >= n8p + nf;
    if (!pad) continue;
    const int sl = qk_slot(pos);
    ws.off[sl] = pos < n8p ? off8 : offf;
    if (pos >= n8p && low_f) atomicOr(&ws.low[sl >> 5], 1u << (sl & 31));
#pragma unroll
    for (int j = 0; j < G; ++j) {
      ws.qrep[j][sl] = 0u;
      if (G > 1) ws.hm[j][sl] = make_uint2(0xFFFFFFFFu, 0u);
    }
  }
  if (lane == 0) {
    ws.n8p = n8p;
    ws.nlist = nlp;
    ws.unit = u;
  }
  __syncwarp();
}

// Scale, store and summarise one page's scores.  After the half-warp fold
// every lane holds the totals of tokens 16*l16 .. +15; lane (half h) finishes
// tokens 16*l16 + 8h .. +7.  A 32-token chunk = lanes {2c, 2c+1} x both halves.
__device__ __forceinline__ void qk_finish(const float* raw, int tok0, int n, float* scores_h, float* stats_h,
                                          float isd) {
  const int lane = threadIdx.x & 31;
  const int nv = min(max(n - tok0, 0), 8);
  float sv[8];
  float m = -INFINITY;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    sv[e] = raw[e] * isd;
    if (e < nv) m = fmaxf(m, sv[e]);
  }
  m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, 1));
  m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, 16));
  float l = 0.f;  // MUFU exp2 of (s - m) log2(e), as in k5_finish
#pragma unroll
  for (int e = 0; e < 8; ++e)
    if (e < nv) {
      float ex;
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(ex) : "f"((sv[e] - m) * 1.4426950408889634f));
      l += ex;
    }
  l += __shfl_xor_sync(0xFFFFFFFFu, l, 1);
  l += __shfl_xor_sync(0xFFFFFFFFu, l, 16);
  float* out = scores_h + tok0;
  if (nv == 8) {
    reinterpret_cast<float4*>(out)[0] = make_float4(sv[0], sv[1], sv[2], sv[3]);
    reinterpret_cast<float4*>(out)[1] = make_float4(sv[4], sv[5], sv[6], sv[7]);
  } else {
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (e < nv) out[e] = sv[e];
  }
  if ((lane & 17) == 0 && tok0 < n) {  // lanes 2c of half 0 own chunk c
    float* ps = stats_h + (tok0 >> 5) * 2;
    ps[0] = m;
    ps[1] = l;
  }
}

template <int G, bool TRUNC>
__global__ void __launch_bounds__(32 * QK_WARPS, QkShape<G>::MINB) qk_kernel(akv_store_t s, akv_cfg_t cfg,
                                                                             akv_step_t st, int cap, float isd,
                                                                             int npg_max) {
  pdl_trigger();
  pdl_wait();
  constexpr int HG = QkShape<G>::HG;
  extern __shared__ __align__(16) uint8_t qk_smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = lane >> 4, l16 = lane & 15;
  QkWarp<G>& ws = reinterpret_cast<QkWarp<G>*>(qk_smem_raw)[warp];
  if (lane == 0) ws.unit = -1;
  __syncwarp();
  const uint64_t pol = evict_first_policy();
  uint32_t tkm = 0xFFFFFFFFu, tf = 0u;
  if (TRUNC) {
    const int kb = cfg.trunc_bits - 6;
    const uint32_t km = (0xFFFFu << (10 - kb)) & 0xFFFFu;
    const uint32_t fill = kb < 10 ? (1u << (9 - kb)) : 0u;
    tkm = km | (km << 16);
    tf = fill | (fill << 16);
  }
  // balanced contiguous item range of this warp
  const long long total = (long long)s.n_units * npg_max;
  const long long nw = (long long)gridDim.x * QK_WARPS, gw = (long long)blockIdx.x * QK_WARPS + warp;
  const long long i0 = total * gw / nw, i1 = total * (gw + 1) / nw;
  const int cap_chunks = s.max_pages * (P / 32);
  UnitPages up;
  up.u = -1;
  up.n = 0;

  // (unit, page) walked incrementally (no 64-bit division per item); the pages past a
  // unit's length are skipped as a block
  int u = (int)(i0 / npg_max), pg = (int)(i0 % npg_max);
  for (long long item = i0; item < i1; item = item + 1, pg = pg + 1 == npg_max ? 0 : pg + 1, u += pg == 0) {
    if (u != up.u) unit_pages_fetch(up, s, u);
    const int n = up.n;
    if (pg * P >= n) {  // rest of this unit is past its length
      item += npg_max - 1 - pg;
      pg = npg_max - 1;
      continue;
    }
    if (ws.unit != u || pg == 0) k_prologue<G, TRUNC>(ws, s, cfg, st, u, n, pg == 0);
    const uint8_t* base = s.k_pool + unit_page(up, s, pg) * PAGE;
    const int nb8 = ws.n8p >> 3, nb = ws.nlist >> 3;

#pragma unroll 1
    for (int j0 = 0; j0 < G; j0 += HG) {
      float acc[HG][16];
#pragma unroll
      for (int jj = 0; jj < HG; ++jj)
#pragma unroll
        for (int e = 0; e < 16; ++e) acc[jj][e] = 0.f;

      // software pipeline over homogeneous batches (T8 batches, then T12/T16
      // batches): the next two batches are in flight while one is computed
      KBatch X[3];
      auto load = [&](int b, KBatch& B) { k_load<G>(B, ws, b, b >= nb8, base, l16, half, pol); };
      auto comp = [&](int b, const KBatch& B) {
        if (G > 1 || b >= nb8) k_compute<HG, true, TRUNC, G>(B, ws, b, half, j0, acc, tkm, tf);
        else k_compute<HG, false, TRUNC, G>(B, ws, b, half, j0, acc, tkm, tf);  // G = 1: lighter T8 rebuild
      };
      if (nb > 0) load(0, X[0]);
      if (nb > 1) load(1, X[1]);
      int b = 0;
      for (; b + 3 <= nb; b += 3) {
        load(b + 2, X[2]);
        comp(b, X[0]);
        if (b + 3 < nb) load(b + 3, X[0]);
        comp(b + 1, X[1]);
        if (b + 4 < nb) load(b + 4, X[1]);
        comp(b + 2, X[2]);
      }
      if (b < nb) comp(b, X[0]);
      if (b + 1 < nb) comp(b + 1, X[1]);

#pragma unroll
      for (int jj = 0; jj < HG; ++jj) {
        float mine[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {  // fold the two half-warps; keep this lane's 8 tokens
          const float lo = acc[jj][e] + __shfl_xor_sync(0xFFFFFFFFu, acc[jj][e], 16);
          const float hi = acc[jj][e + 8] + __shfl_xor_sync(0xFFFFFFFFu, acc[jj][e + 8], 16);
          mine[e] = half ? hi : lo;
        }
        const size_t hh = (size_t)u * G + j0 + jj;
        qk_finish(mine, pg * P + 16 * l16 + 8 * half, n, st.scores + hh * cap, st.page_stats + hh * cap_chunks * 2,
                  isd);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// qk v5 (GQA groups, G = 4 / 8): tensor-core scores from a per-warp cp.async ring.
//
// The G q-heads of a unit share every K tile, so a page is a small GEMM:
// scores[256 tokens][G] = K~^T[256][channels] x Q[channels][G], issued as
// mma.sync m16n8k8 (fp16 in, fp32 accumulate: products exact, D9) with the
// heads on N (G <= 8).  Per-head tiers differ per channel, so K~ is split by
// tier variant: a chunk's words are rebuilt once at the union tier and masked
// down to T12 / T8 (midpoint fill), and each variant is multiplied by the q
// fragment that holds only the heads of that tier (zero elsewhere):
//   s_j = sum_c q_jc K~_{tier_j(c)}(c) = sum_v K~_v . (q_j masked to tier v).
// The channel order inside the reduction is free, so list positions map
// straight onto the mma K index: lane (g, t) holds positions 2t, 2t+1 of an
// 8-channel chunk for tokens 16g..16g+15 and 128+16g..+15; m16 tile i < 8
// takes tokens 16g+2i (row g) and 16g+2i+1 (row g+8) of the first page half,
// tiles 8..15 the same in the second half.
//
// With the math this light the kernel is bound by how many bytes are in
// flight (DRAM latency under load is several us), so the rows are staged by
// 16-byte cp.async into a ring of 4 KB slots per warp, NB-1 slots ahead of the
// math and continuous across the pages of a unit: a slot is 16 T8-class head
// rows, or 8 T12/T16-class head rows + their mid rows (+ low rows for T16).
// Shared-memory reads are bank-conflict free: head rows are read as 4 rows x
// 128 B per LDS.128; the 128 B nibble rows are stored with their 64 B halves
// swapped on every other row pair.
// ---------------------------------------------------------------------------
#ifndef AKV_QK5_NB4
#define AKV_QK5_NB4 3
#endif
#ifndef AKV_QK5_MINB4
#define AKV_QK5_MINB4 3
#endif
constexpr int Q5_SLOT = 4096;
constexpr int Q5_CHUNKS = 18;  // (128 + 15 + 7) / 8 eight-channel chunks: T8 class padded to 16, T12/T16 class to 8

template <int G>
struct alignas(16) Qk5Warp {
  uint32_t off[Q5_CHUNKS * 8];            // list position -> channel * P
  // per chunk, tier variant (T8, T12, T16), lane (g, t): the B fragment; G <= 4 keeps only
  // the lanes of heads g < 4 (lanes 0..15; the padding heads' fragments are zero)
  uint32_t bf[Q5_CHUNKS][3][G <= 4 ? 16 : 32];
  uint32_t low[(Q5_CHUNKS * 8 + 31) / 32];  // list position bitmask: low row needed (T16 in the union)
  uint8_t vmask[Q5_CHUNKS];               // variants present per chunk (bit 0 T8, 1 T12, 2 T16)
  int n8p, nlp, unit, pad;
};

template <int G>
__device__ __forceinline__ uint32_t q5_bfrag(const Qk5Warp<G>& ws, int c, int v) {
  const int lane = threadIdx.x & 31;
  if (G <= 4) return lane < 16 ? ws.bf[c][v][lane] : 0u;
  return ws.bf[c][v][lane];
}

template <int G>
struct Qk5Shape {
  static constexpr int WARPS = 4;
  // G = 4: 3 ring slots and 168 registers -> 3 CTAs (12 warps) per SM; G = 8: 5 slots, 2 CTAs
  static constexpr int NB = G <= 4 ? AKV_QK5_NB4 : 5;  // ring slots per warp
  static constexpr int LIST = (sizeof(Qk5Warp<G>) + 127) & ~127;
  static constexpr int PER_WARP = LIST + NB * Q5_SLOT + 128;  // list | ring | slot mbarriers (TMA staging)
  static constexpr int SMEM = WARPS * PER_WARP;
  static constexpr int MINB = G <= 4 ? AKV_QK5_MINB4 : 2;
  static_assert(G * Q5_CHUNKS * 8 * 3 <= NB * Q5_SLOT, "prologue scratch must fit the ring");
};

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Rule 1 + lists, B fragments and variant masks.  Runs with the ring drained
// (its memory holds the per-position q / code scratch).
template <int G, bool TRUNC>
__device__ void k5_prologue(Qk5Warp<G>& ws, uint8_t* scratch, const akv_store_t& s, const akv_cfg_t& cfg,
                            const akv_step_t& st, int u, int n, bool book) {
  const int lane = threadIdx.x & 31;
  uint16_t(*qh)[Q5_CHUNKS * 8] = reinterpret_cast<uint16_t(*)[Q5_CHUNKS * 8]>(scratch);
  uint8_t(*cd)[Q5_CHUNKS * 8] = reinterpret_cast<uint8_t(*)[Q5_CHUNKS * 8]>(scratch + G * Q5_CHUNKS * 8 * 2);
  uint32_t qw[G][4];
  int code[G][4], ucode[4];
  k_rule1<G, TRUNC>(s, cfg, st, u, n, book, qw, code, ucode);
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t b8[4], bf[4];
  int n8 = 0, nf = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    b8[k] = __ballot_sync(0xFFFFFFFFu, ucode[k] == 8);
    bf[k] = __ballot_sync(0xFFFFFFFFu, ucode[k] >= 12);
    n8 += __popc(b8[k]);
    nf += __popc(bf[k]);
  }
  // at least one slot per page, so an all-SKIP unit still writes its (zero) scores
  const int n8p = (n8 + nf == 0) ? 16 : (n8 + 15) & ~15, nlp = n8p + ((nf + 7) & ~7);
  // pads: channel 0's rows, q = 0, code 0
  for (int pos = lane; pos < Q5_CHUNKS * 8; pos += 32) {
    ws.off[pos] = 0u;
#pragma unroll
    for (int j = 0; j < G; ++j) {
      qh[j][pos] = 0;
      cd[j][pos] = 0;
    }
  }
  if (lane < (Q5_CHUNKS * 8 + 31) / 32) ws.low[lane] = 0u;
  __syncwarp();
  int base8 = 0, basef = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int c = lane + 32 * k;
    int pos = -1;
    if (ucode[k] == 8) pos = base8 + __popc(b8[k] & lt);
    else if (ucode[k] >= 12) pos = n8p + basef + __popc(bf[k] & lt);
    if (pos >= 0) {
      ws.off[pos] = (uint32_t)c * P;
      if (ucode[k] == 16) atomicOr(&ws.low[pos >> 5], 1u << (pos & 31));
#pragma unroll
      for (int j = 0; j < G; ++j) {
        qh[j][pos] = code[j][k] ? (uint16_t)(qw[j][k] & 0xFFFFu) : (uint16_t)0;
        cd[j][pos] = (uint8_t)code[j][k];
      }
    }
    base8 += __popc(b8[k]);
    basef += __popc(bf[k]);
  }
  __syncwarp();
  // B fragments: lane (g, t) holds head g's q at list positions 2t, 2t+1 of the chunk
  const int g = lane >> 2, t = lane & 3;
  const int nch = nlp >> 3, n8c = n8p >> 3;
  for (int c = 0; c < nch; ++c) {
    const int p0 = c * 8 + 2 * t;
    uint32_t q0 = 0u, q1 = 0u, c0 = 0u, c1 = 0u;
    if (g < G) {
      q0 = qh[g][p0];
      q1 = qh[g][p0 + 1];
      c0 = cd[g][p0];
      c1 = cd[g][p0 + 1];
    }
    uint32_t vm = 0u;
#pragma unroll
    for (int v = 0; v < 3; ++v) {
      const uint32_t tier = 8u + 4u * v;
      const uint32_t b = (c0 == tier ? q0 : 0u) | ((c1 == tier ? q1 : 0u) << 16);
      if (G > 4 || lane < 16) ws.bf[c][v][lane & (G <= 4 ? 15 : 31)] = b;
      if (__any_sync(0xFFFFFFFFu, b != 0u)) vm |= 1u << v;
    }
    if (lane == 0) ws.vmask[c] = (uint8_t)(c < n8c ? 1u : vm);
  }
  if (lane == 0) {
    ws.n8p = n8p;
    ws.nlp = nlp;
    ws.unit = u;
  }
  __syncwarp();
}

// Copy slot b of a page into the ring (one commit group).
template <int G>
__device__ __forceinline__ void q5_issue(uint8_t* slot, const Qk5Warp<G>& ws, int b, const uint8_t* base) {
  const int lane = threadIdx.x & 31;
  const int n8s = ws.n8p >> 4;
  if (b < n8s) {
    const int p0 = 16 * b;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int idx = lane + 32 * k, r = idx >> 4, col = idx & 15;
      cp_async16(slot + r * 256 + col * 16, base + ws.off[p0 + r] + col * 16);
    }
  } else {
    const int p0 = ws.n8p + 8 * (b - n8s);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int idx = lane + 32 * k, r = idx >> 4, col = idx & 15;
      cp_async16(slot + r * 256 + col * 16, base + ws.off[p0 + r] + col * 16);
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int idx = lane + 32 * k, r = idx >> 3, col = idx & 7;
      const int pos = p0 + r;
      const uint8_t* src = base + MID + (ws.off[pos] >> 1) + col * 16;
      uint8_t* dst = slot + 2048 + r * 128 + ((col ^ (((r >> 1) & 1) << 2)) << 4);
      cp_async16(dst, src);
      if ((ws.low[pos >> 5] >> (pos & 31)) & 1u) cp_async16(dst + 1024, src + (LOW - MID));
    }
  }
  cp_async_commit();
}

// 2-D TMA gather of four rows (UTMALDG.2D.GATHER4): rows r0..r3 of the map, column 0, into
// four consecutive rows at dst.
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* tm, int r0, int r1, int r2, int r3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
      "%6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}

// Slot b of a page by TMA gathers (lane 0): the K pool as rows of 256 B (t256: head rows,
// channel c of page pid = row 256 pid + c) and of 128 B (t128: mid row = 512 pid + 256 + c,
// low row = 512 pid + 384 + c).  A slot's positions without a low row gather their own mid
// row again instead (an L2 hit: no extra DRAM bytes; the word is not used).
template <int G>
__device__ __forceinline__ void q5_issue_tma(uint8_t* slot, uint64_t* bar, const Qk5Warp<G>& ws, int b, long long pid,
                                             const CUtensorMap* t256, const CUtensorMap* t128) {
  const int n8s = ws.n8p >> 4;
  const int h0 = (int)(pid * 256), m0 = (int)(pid * 512) + 256;
  if (b < n8s) {
    const int p0 = 16 * b;
    mbar_arrive_expect_tx(bar, 4096);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 o = *reinterpret_cast<const uint4*>(&ws.off[p0 + 4 * q]);
      tma_gather4(slot + q * 1024, t256, h0 + (int)(o.x >> 8), h0 + (int)(o.y >> 8), h0 + (int)(o.z >> 8),
                  h0 + (int)(o.w >> 8), bar);
    }
  } else {
    const int p0 = ws.n8p + 8 * (b - n8s);
    const uint32_t lowm = (ws.low[p0 >> 5] >> (p0 & 31)) & 0xFFu;
    mbar_arrive_expect_tx(bar, 4096);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const uint4 o = *reinterpret_cast<const uint4*>(&ws.off[p0 + 4 * q]);
      const int c0 = (int)(o.x >> 8), c1 = (int)(o.y >> 8), c2 = (int)(o.z >> 8), c3 = (int)(o.w >> 8);
      tma_gather4(slot + q * 1024, t256, h0 + c0, h0 + c1, h0 + c2, h0 + c3, bar);
      tma_gather4(slot + 2048 + q * 512, t128, m0 + c0, m0 + c1, m0 + c2, m0 + c3, bar);
      const uint32_t lm = lowm >> (4 * q);
      tma_gather4(slot + 3072 + q * 512, t128, m0 + c0 + ((lm & 1u) ? 128 : 0), m0 + c1 + ((lm & 2u) ? 128 : 0),
                  m0 + c2 + ((lm & 4u) ? 128 : 0), m0 + c3 + ((lm & 8u) ? 128 : 0), bar);
    }
  }
}

struct K5Head {
  uint4 h[2][2];  // [channel][page half]: 16 tokens each
};
struct K5Nib {
  uint2 m[2][2], l[2][2];
};

__device__ __forceinline__ uint32_t u4w(const uint4& v, int i) {
  return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

__device__ __forceinline__ void mma_f16_1688(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t b) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(b));
}

// (x & m) | f as one LOP3 with both constants in registers
__device__ __forceinline__ uint32_t mask_fill(uint32_t x, uint32_t m, uint32_t f) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(x), "r"(m), "r"(f));
  return r;
}

__device__ __forceinline__ void k5_compute_t8(const K5Head& X, uint32_t b8, float (&acc)[16][4], uint32_t c80) {
#pragma unroll
  for (int hf = 0; hf < 2; ++hf)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      // token 16g + 2i (of the half) is byte 2i of the lane's 16 head bytes of each channel
      const int wi = i >> 1, p = 2 * (i & 1);
      // x = (ch0 token 2i, ch0 token 2i+1, ch1 token 2i, ch1 token 2i+1), then the head
      // bytes into positions 1 and 3 with the 0x80 midpoint fill in 0 and 2
      const uint32_t x = prmt(u4w(X.h[0][hf], wi), u4w(X.h[1][hf], wi), (uint32_t)(((5 + p) << 12) | ((4 + p) << 8) |
                                                                                       ((p + 1) << 4) | p));
      mma_f16_1688(acc[8 * hf + i], prmt(x, c80, 0x2404), prmt(x, c80, 0x3414), b8);
    }
}

// vm: the tier variants present in the chunk (bit 0 T8, 1 T12, 2 T16).  The words are
// rebuilt once at the union tier; each present variant is one warp-uniform branch over
// the 16 tiles (no predicated-off mma; specialising every combination as a template
// was slower: code growth, profiles/r01_history.md #32).
template <bool TRUNC>
__device__ __forceinline__ void k5_compute_full(const K5Head& X, const K5Nib& N, uint32_t vm, uint32_t b8,
                                                uint32_t b12, uint32_t b16, float (&acc)[16][4], uint32_t tkm,
                                                uint32_t tf, uint32_t c80) {
  uint32_t A[16][2];
#pragma unroll
  for (int hf = 0; hf < 2; ++hf)
#pragma unroll
    for (int hv = 0; hv < 2; ++hv) {  // tokens 8hv .. 8hv+7 of the lane's 16 in this half
      uint32_t W[2][4];  // per channel: token pairs (2k, 2k+1) at the union tier
#pragma unroll
      for (int j = 0; j < 2; ++j)
        assemble8(hv ? X.h[j][hf].z : X.h[j][hf].x, hv ? X.h[j][hf].w : X.h[j][hf].y,
                  hv ? N.m[j][hf].y : N.m[j][hf].x, hv ? N.l[j][hf].y : N.l[j][hf].x, W[j]);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int i = 8 * hf + 4 * hv + k;
        A[i][0] = prmt(W[0][k], W[1][k], 0x5410);
        A[i][1] = prmt(W[0][k], W[1][k], 0x7632);
        if (TRUNC) {
          A[i][0] = mask_fill(A[i][0], tkm, tf);
          A[i][1] = mask_fill(A[i][1], tkm, tf);
        }
      }
    }
  if (vm & 4u) {
#pragma unroll
    for (int i = 0; i < 16; ++i) mma_f16_1688(acc[i], A[i][0], A[i][1], b16);
  }
  if (vm & 2u) {
    uint32_t m12 = 0xFFF0FFF0u, f12 = 0x00080008u;
    asm volatile("" : "+r"(m12), "+r"(f12));  // mask / fill in registers: one LOP3 per word
#pragma unroll
    for (int i = 0; i < 16; ++i)
      mma_f16_1688(acc[i], mask_fill(A[i][0], m12, f12), mask_fill(A[i][1], m12, f12), b12);
  }
  if (vm & 1u) {
#pragma unroll
    for (int i = 0; i < 16; ++i) mma_f16_1688(acc[i], prmt(A[i][0], c80, 0x3414), prmt(A[i][1], c80, 0x3414), b8);
  }
}

template <int G, bool TRUNC, bool TMAQ>
__device__ __forceinline__ void q5_compute(const uint8_t* slot, const Qk5Warp<G>& ws, int b, float (&acc)[16][4],
                                           uint32_t tkm, uint32_t tf, uint32_t c80) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int n8s = ws.n8p >> 4;
  if (b < n8s) {
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
      K5Head X;
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int hf = 0; hf < 2; ++hf)
          X.h[j][hf] = *reinterpret_cast<const uint4*>(slot + (8 * cc + 2 * t + j) * 256 + 128 * hf + 16 * g);
      k5_compute_t8(X, q5_bfrag<G>(ws, 2 * b + cc, 0), acc, c80);
    }
  } else {
    const int ch = (ws.n8p >> 3) + (b - n8s), p0 = ws.n8p + 8 * (b - n8s) + 2 * t;
    const uint32_t lowm = (ws.low[p0 >> 5] >> (p0 & 31)) & 3u;
    K5Head X;
    K5Nib N;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int r = 2 * t + j;
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        X.h[j][hf] = *reinterpret_cast<const uint4*>(slot + r * 256 + 128 * hf + 16 * g);
        const int nb = 2048 + r * 128 + (TMAQ ? 64 * hf + 8 * g : ((64 * hf + 8 * g) ^ ((t & 1) << 6)));
        N.m[j][hf] = *reinterpret_cast<const uint2*>(slot + nb);
        N.l[j][hf] = ((lowm >> j) & 1u) ? *reinterpret_cast<const uint2*>(slot + nb + 1024)
                                        : make_uint2(0x88888888u, 0x88888888u);
      }
    }
    const uint32_t b8 = q5_bfrag<G>(ws, ch, 0), b12 = q5_bfrag<G>(ws, ch, 1), b16 = q5_bfrag<G>(ws, ch, 2);
    k5_compute_full<TRUNC>(X, N, ws.vmask[ch], b8, b12, b16, acc, tkm, tf, c80);
  }
}

// Scale, store and summarise one head's 16 tokens (16g .. 16g+15 of a page half);
// a 32-token chunk = lanes g = 2c, 2c+1 (lane ^ 4).
__device__ __forceinline__ void k5_finish(const float (&raw)[16], int tok0, int n, float* scores_h, float* stats_h,
                                          float isd, bool store) {
  const int lane = threadIdx.x & 31;
  const int nv = min(max(n - tok0, 0), 16);
  float sv[16];
  float m = -INFINITY;
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    sv[e] = raw[e] * isd;
    if (e < nv) m = fmaxf(m, sv[e]);
  }
  m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, 4));
  // sum of exp(s - m) over <= 32 terms by the MUFU exp2 (rel. error ~2^-22 per term: L and
  // every p move by ~1e-7 relative).  s - m is formed first so the maximum term is exactly
  // ex2(0) = 1 (a one-hot softmax stays exactly one-hot).
  float l = 0.f;
#pragma unroll
  for (int e = 0; e < 16; ++e)
    if (e < nv) {
      float ex;
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(ex) : "f"((sv[e] - m) * 1.4426950408889634f));
      l += ex;
    }
  l += __shfl_xor_sync(0xFFFFFFFFu, l, 4);
  if (!store) return;  // (lanes of absent heads: the shuffles above need the whole warp)
  float* out = scores_h + tok0;
  if (nv == 16) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      reinterpret_cast<float4*>(out)[q] = make_float4(sv[4 * q], sv[4 * q + 1], sv[4 * q + 2], sv[4 * q + 3]);
  } else {
#pragma unroll
    for (int e = 0; e < 16; ++e)
      if (e < nv) out[e] = sv[e];
  }
  if (((lane >> 2) & 1) == 0 && tok0 < n) {  // even g owns the chunk
    float* ps = stats_h + (tok0 >> 5) * 2;
    ps[0] = m;
    ps[1] = l;
  }
}

template <int G, bool TRUNC, bool TMAQ>
__global__ void __launch_bounds__(32 * Qk5Shape<G>::WARPS, Qk5Shape<G>::MINB)
    qk5_kernel(akv_store_t s, akv_cfg_t cfg, akv_step_t st, int cap, float isd, int npg_max,
               const __grid_constant__ CUtensorMap t256, const __grid_constant__ CUtensorMap t128) {
  using S = Qk5Shape<G>;
  constexpr int NB = S::NB;
  pdl_trigger();
  pdl_wait();
  extern __shared__ __align__(128) uint8_t qk5_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  Qk5Warp<G>& ws = *reinterpret_cast<Qk5Warp<G>*>(qk5_smem + warp * S::PER_WARP);
  uint8_t* ring = qk5_smem + warp * S::PER_WARP + S::LIST;
  uint64_t* sbar = reinterpret_cast<uint64_t*>(ring + NB * Q5_SLOT);  // TMAQ: one mbarrier per slot
  if (TMAQ) {
    if (lane == 0) {
      for (int i = 0; i < NB; ++i) mbar_init(&sbar[i], 1);
      mbar_fence_init();
    }
    __syncwarp();
  }
  uint32_t sphase = 0u;  // TMAQ: parity bit per slot
  uint32_t tkm = 0xFFFFFFFFu, tf = 0u, c80 = 0x80808080u;
  asm volatile("" : "+r"(c80));
  if (TRUNC) {
    const int kb = cfg.trunc_bits - 6;
    const uint32_t km = (0xFFFFu << (10 - kb)) & 0xFFFFu;
    const uint32_t fill = kb < 10 ? (1u << (9 - kb)) : 0u;
    tkm = km | (km << 16);
    tf = fill | (fill << 16);
  }
  // balanced contiguous range of (unit, page) items
  const long long total = (long long)s.n_units * npg_max;
  const long long nw = (long long)gridDim.x * S::WARPS, gw = (long long)blockIdx.x * S::WARPS + warp;
  const long long i0 = total * gw / nw, i1 = total * (gw + 1) / nw;
  const int cap_chunks = s.max_pages * (P / 32);

  // load cursor (l, lb) and compute cursor (c, cb) over (item, slot); both walk the same
  // items, (unit, page) advanced incrementally (no 64-bit division per page)
  struct Cur {
    long long i;
    int u, pg;
  };
  UnitPages lup, cup;
  lup.u = cup.u = -1;
  lup.n = cup.n = 0;
  auto seek = [&](Cur& c, UnitPages& up) {  // first valid item at or after c
    while (c.i < i1) {
      if (c.u != up.u) unit_pages_fetch(up, s, c.u);
      if (c.pg * P < up.n) return;
      c.i += npg_max - c.pg;  // the rest of this unit is past its length
      c.pg = 0;
      ++c.u;
    }
  };
  auto advance = [&](Cur& c, UnitPages& up) {
    ++c.i;
    if (++c.pg == npg_max) {
      c.pg = 0;
      ++c.u;
    }
    seek(c, up);
  };
  Cur lc{i0, (int)(i0 / npg_max), (int)(i0 % npg_max)};
  seek(lc, lup);
  Cur cc = lc;
  cup = lup;
  int lb = 0, cb = 0, issued = 0, computed = 0, islot = 0, cslot = 0;
  bool lblocked = false;  // the load cursor reached a unit whose lists are not built yet
  const uint8_t* lbase = nullptr;
  long long lpid = 0;
  if (lc.i < i1) {
    k5_prologue<G, TRUNC>(ws, ring, s, cfg, st, lc.u, lup.n, lc.pg == 0);
    lpid = (long long)unit_page(lup, s, lc.pg);
    lbase = s.k_pool + lpid * PAGE;
  }
  float acc[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;

  // One cp.async group is committed per step (an empty one when the load cursor waits at a
  // unit boundary), so the slot about to be computed always has NB-2 groups after it and a
  // constant wait_group<NB-2> suffices.
  auto issue_one = [&]() {
    if (lc.i < i1 && !lblocked) {
      const int nslots = (ws.n8p >> 4) + ((ws.nlp - ws.n8p) >> 3);
      if (TMAQ) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads / scratch before async writes
        if (lane == 0) q5_issue_tma<G>(ring + islot * Q5_SLOT, &sbar[islot], ws, lb, lpid, &t256, &t128);
      } else {
        q5_issue<G>(ring + islot * Q5_SLOT, ws, lb, lbase);
      }
      ++issued;
      islot = islot + 1 == NB ? 0 : islot + 1;
      if (++lb == nslots) {
        lb = 0;
        const int pu = lc.u;
        advance(lc, lup);
        if (lc.i < i1) {
          if (lc.u != pu) {
            lblocked = true;  // new unit: wait for the math to drain
          } else {
            lpid = (long long)unit_page(lup, s, lc.pg);
            lbase = s.k_pool + lpid * PAGE;
          }
        }
      }
    } else if (!TMAQ) {
      cp_async_commit();
    }
  };
#pragma unroll 1
  for (int k = 0; k < NB - 1; ++k) issue_one();
  while (cc.i < i1) {
    const int nslots = (ws.n8p >> 4) + ((ws.nlp - ws.n8p) >> 3);
    if (issued == computed) {
      // drained at a unit boundary: build the next unit's lists, refill the ring
      k5_prologue<G, TRUNC>(ws, ring, s, cfg, st, lc.u, lup.n, lc.pg == 0);
      lpid = (long long)unit_page(lup, s, lc.pg);
      lbase = s.k_pool + lpid * PAGE;
      lblocked = false;
#pragma unroll 1
      for (int k = 0; k < NB - 1; ++k) issue_one();
      continue;
    }
    if (TMAQ) {
      mbar_wait(&sbar[cslot], (sphase >> cslot) & 1u);
      sphase ^= 1u << cslot;
    } else {
      cp_async_wait<NB - 2>();
    }
    __syncwarp();
    q5_compute<G, TRUNC, TMAQ>(ring + cslot * Q5_SLOT, ws, cb, acc, tkm, tf, c80);
    ++computed;
    cslot = cslot + 1 == NB ? 0 : cslot + 1;
    __syncwarp();  // every lane is done with the slot before it is refilled
    issue_one();
    if (++cb == nslots) {
      // page done: lane (g, t) holds tokens 16g + 2i (acc[i][0..1]) and 16g + 2i + 1
      // (acc[i][2..3]) of each page half for heads 2t, 2t+1
      const int u = cc.u, pg = cc.pg;
      const int n = cup.n;
      if (G == 4) {
        // heads 4..7 are padding: lanes t >= 2 take over page half 1 of lane t - 2, so
        // every lane finishes 2 x 16 values instead of 4 x 16
        const int hfe = t >> 1, src = t >= 2 ? lane - 2 : lane;
        float mine[8][4];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float v = __shfl_sync(0xFFFFFFFFu, acc[8 + i][e], src);
            mine[i][e] = hfe ? v : acc[i][e];
          }
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          float raw[16];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            raw[2 * i] = mine[i][hh];
            raw[2 * i + 1] = mine[i][2 + hh];
          }
          const size_t h = (size_t)u * G + 2 * (t & 1) + hh;
          k5_finish(raw, pg * P + 128 * hfe + 16 * g, n, st.scores + h * cap, st.page_stats + h * cap_chunks * 2,
                    isd, true);
        }
      } else {
#pragma unroll
        for (int hf = 0; hf < 2; ++hf)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            float raw[16];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              raw[2 * i] = acc[8 * hf + i][hh];
              raw[2 * i + 1] = acc[8 * hf + i][2 + hh];
            }
            const int j = 2 * t + hh;
            const size_t h = (size_t)u * G + (j < G ? j : 0);
            k5_finish(raw, pg * P + 128 * hf + 16 * g, n, st.scores + h * cap, st.page_stats + h * cap_chunks * 2,
                      isd, j < G);
          }
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
      cb = 0;
      advance(cc, cup);
    }
  }
}

}  // namespace akv

#include "akv_qk8.cuh"
#include "akv_qk9.cuh"

namespace akv {

// AKV_QK5_TMA=1 stages qk5's slots by TMA gathers (four channel rows per
// UTMALDG.2D.GATHER4, parity-green) instead of 16-byte cp.async: measured slower at c3
// (qk 144.5 vs 133.1 us, profiles/r02_history.md r2-4), so the default stays cp.async.
template <int G, bool TRUNC>
static void launch_qk5_t(const akv_store_t& s, const akv_cfg_t& cfg, const akv_step_t& st, int max_len,
                         cudaStream_t stream) {
  using S = Qk5Shape<G>;
  static const int use_tma = env_int("AKV_QK5_TMA", 0);
  const unsigned long long pages = s.pool_pages > 0 ? (unsigned long long)s.pool_pages
                                                    : (unsigned long long)s.n_units * s.max_pages;
  CUtensorMap t256, t128;
  const bool tma = use_tma && tmap_2d(s.k_pool, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, 256, pages * 256, 256, 1,
                                      CU_TENSOR_MAP_SWIZZLE_NONE, &t256) &&
                   tmap_2d(s.k_pool, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, 128, pages * 512, 128, 1,
                           CU_TENSOR_MAP_SWIZZLE_NONE, &t128);
  const int cap = s.max_pages * P;
  const int npg = (max_len + P - 1) / P;
  const long long items = (long long)s.n_units * npg;
  const float isd = (float)(1.0 / 11.313708498984761);  // 1/sqrt(128)
  if (tma) {
    const int resident = resident_ctas<qk5_kernel<G, TRUNC, true>>(32 * S::WARPS, S::SMEM);
    const int grid = (int)std::min<long long>(resident, std::max<long long>((items + S::WARPS - 1) / S::WARPS, 1));
    launch_pdl(PDL_QK, qk5_kernel<G, TRUNC, true>, dim3(grid), dim3(32 * S::WARPS), (size_t)S::SMEM, stream, s, cfg, st, cap,
               isd, npg, t256, t128);
    return;
  }
  const int resident = resident_ctas<qk5_kernel<G, TRUNC, false>>(32 * S::WARPS, S::SMEM);
  const int grid = balanced_grid(items, resident, S::WARPS);
  launch_pdl(PDL_QK, qk5_kernel<G, TRUNC, false>, dim3(grid), dim3(32 * S::WARPS), (size_t)S::SMEM, stream, s, cfg, st, cap, isd,
             npg, t256, t128);
}

// G <= 2: the direct-load FHFMA kernel; G >= 4: the mma.sync ring kernel qk5 (one K tile
// feeds 4-8 heads, so the FHFMA path would be issue bound).  AKV_QK_KERNEL=qk9 selects the
// tcgen05 / TMEM kernel (parity-green, slower at c3: profiles/r02_history.md r2-7).
// AKV_QK_KERNEL=tma selects qk8 (the per-warp bulk-copy ring, akv_qk8.cuh) for A/B
// measurements; the default is the direct-load kernel for G <= 2 and qk5 for G >= 4
// (measured faster: profiles/r02_qk_tma_vs_ldg.md).
static int qk_choice() {
  static const int v = [] {
    const char* e = getenv("AKV_QK_KERNEL");
    if (e && strcmp(e, "tma") == 0) return 8;
    if (e && strcmp(e, "qk9") == 0) return 9;
    return 0;
  }();
  return v;
}
static bool qk_tma() { return qk_choice() == 8; }

template <int G, bool TRUNC>
static void launch_qk_t(const akv_store_t& s, const akv_cfg_t& cfg, const akv_step_t& st, int max_len,
                        cudaStream_t stream) {
  if (qk_tma()) {
    launch_qk8_t<G, TRUNC>(s, cfg, st, max_len, stream);
  } else if constexpr (G >= 4) {
    if (qk_choice() == 9) launch_qk9_t<G, TRUNC>(s, cfg, st, max_len, stream);
    else launch_qk5_t<G, TRUNC>(s, cfg, st, max_len, stream);
  } else {
    const size_t smem = sizeof(QkWarp<G>) * QK_WARPS;
    const int resident = resident_ctas<qk_kernel<G, TRUNC>>(32 * QK_WARPS, smem);
    const int cap = s.max_pages * P;
    const int npg = (max_len + P - 1) / P;
    const long long items = (long long)s.n_units * npg;
    const int grid = balanced_grid(items, resident, QK_WARPS);
    const float isd = (float)(1.0 / 11.313708498984761);  // 1/sqrt(128)
    launch_pdl(PDL_QK, qk_kernel<G, TRUNC>, dim3(grid), dim3(32 * QK_WARPS), smem, stream, s, cfg, st, cap, isd, npg);
  }
}

void launch_qk(const akv_store_t& s, const akv_cfg_t& cfg, const akv_step_t& st, int max_len, cudaStream_t stream) {
  const bool tr = cfg.trunc_bits != 0;
  switch (cfg.group) {
    case 1: tr ? launch_qk_t<1, true>(s, cfg, st, max_len, stream) : launch_qk_t<1, false>(s, cfg, st, max_len, stream); break;
    case 2: tr ? launch_qk_t<2, true>(s, cfg, st, max_len, stream) : launch_qk_t<2, false>(s, cfg, st, max_len, stream); break;
    case 4: tr ? launch_qk_t<4, true>(s, cfg, st, max_len, stream) : launch_qk_t<4, false>(s, cfg, st, max_len, stream); break;
    case 8: tr ? launch_qk_t<8, true>(s, cfg, st, max_len, stream) : launch_qk_t<8, false>(s, cfg, st, max_len, stream); break;
  }
}

}  // namespace akv
