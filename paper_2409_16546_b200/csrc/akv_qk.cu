// scores_aligned for every (unit, q-head) of a batch.
//
// Persistent warps pull (unit, page) items from an atomic queue (no wave
// tail; deterministic because each page's result does not depend on which
// warp computes it).  Per item a warp:
//
//  1. evaluates Rule 1 for its unit (rule1_target SPEC.md:157-165,
//     required_mantissa_bits :139-147, tier_for_bits :148-156,
//     k_channel_tiers :175-183) for every q-head
//     of the kv-head, and builds a channel list ordered by union class:
//     T8 channels first (head plane only), then T12/T16 channels; SKIP
//     channels are dropped (0 bits read);
//  2. streams the page: lane = 8 consecutive tokens; per listed channel one
//     LDG.64 of the 256 B head-plane row and, only for T12/T16 channels, one
//     LDG.32 of the 128 B mid row (+ low row for T16).  Loads are
//     software-pipelined one 8-channel batch ahead (ping-pong registers);
//  3. rebuilds fp16 words with PRMT/LOP3 (midpoint fill for absent nibbles,
//     HB:160-179) and accumulates q_c * K~ with the mixed-precision FHFMA
//     (exact fp16 x fp16 products, fp32 sums, D9);
//  4. scales by 1/sqrt(d) after accumulation and writes the
//     page's scores and (max, sum exp) for the split softmax.
#include <algorithm>

#include "akv_common.cuh"

namespace akv {

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

// Per-warp prologue state; lists are in "list order" (T8 class first).
template <int G>
struct alignas(16) QkWarp {
  uint32_t q[G][D / 2];  // q (fp16) per list position, pairs (2p, 2p+1); 0 for SKIP heads / pads
  uint2 hm[G][D];        // per-head (keep, fill) word masks per list position (used when G > 1)
  uint16_t ent[D];       // channel | class << 8 ; class 0 = pad
  int nlist;             // padded to a multiple of 8
  int unit;
};

struct KBatch {
  uint2 h[8];
  uint32_t m[8], l[8];
  uint4 e;  // 8 list entries
};

__device__ __forceinline__ uint32_t ent_of(const uint4& e, int i) {
  const uint32_t w = i < 2 ? e.x : (i < 4 ? e.y : (i < 6 ? e.z : e.w));
  return (i & 1) ? (w >> 16) : (w & 0xFFFFu);
}

template <int G>
__device__ __forceinline__ void k_load(KBatch& X, const QkWarp<G>& ws, int b, const uint8_t* hb, const uint8_t* mb,
                                       uint64_t pol) {
  X.e = *reinterpret_cast<const uint4*>(&ws.ent[b * 8]);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t en = ent_of(X.e, i);
    const uint32_t ch = en & 0xFFu, cls = en >> 8;
    if (cls) X.h[i] = ld_stream_u64(hb + ch * P, pol);
    if (cls >= 12) X.m[i] = ld_stream_u32(mb + ch * (P / 2), pol);
    if (cls == 16) X.l[i] = ld_stream_u32(mb + ch * (P / 2) + (LOW - MID), pol);
  }
}

template <int G, bool TRUNC>
__device__ __forceinline__ void k_compute(const KBatch& X, const QkWarp<G>& ws, int b, float acc[G][8],
                                          uint32_t tkm, uint32_t tf) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t en = ent_of(X.e, i);
    const uint32_t cls = en >> 8;
    if (cls == 0) continue;  // pad (warp-uniform)
    const int pos = b * 8 + i;
    uint32_t w[4];
    if (cls == 8) {
      const uint32_t c80 = 0x80808080u;
      w[0] = prmt(X.h[i].x, c80, 0x1404);
      w[1] = prmt(X.h[i].x, c80, 0x3424);
      w[2] = prmt(X.h[i].y, c80, 0x1404);
      w[3] = prmt(X.h[i].y, c80, 0x3424);
    } else {
      assemble8(X.h[i].x, X.h[i].y, X.m[i], cls == 16 ? X.l[i] : 0x88888888u, w);
    }
    if (TRUNC) {
#pragma unroll
      for (int k = 0; k < 4; ++k) w[k] = (w[k] & tkm) | tf;
    }
#pragma unroll
    for (int j = 0; j < G; ++j) {
      uint32_t wj[4];
      if (G > 1 && cls != 8) {
        const uint2 hm = ws.hm[j][pos];
#pragma unroll
        for (int k = 0; k < 4; ++k) wj[k] = (w[k] & hm.x) | hm.y;
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) wj[k] = w[k];
      }
      const uint32_t qp = ws.q[j][pos >> 1];
      if (i & 1)
        fma8<1>(wj, qp, acc[j]);
      else
        fma8<0>(wj, qp, acc[j]);
    }
  }
}

// Rule 1 for unit u, all G heads; builds the warp's channel list.
template <int G, bool TRUNC>
__device__ void k_prologue(QkWarp<G>& ws, const akv_store_t& s, const akv_cfg_t& cfg, const akv_step_t& st, int u,
                           int n, bool book) {
  const int lane = threadIdx.x & 31;
  const bool aligned = cfg.force_tier == 0 && !TRUNC;
  uint32_t cm[4], qw[G][4];
  int code[G][4], ucode[4] = {0, 0, 0, 0};
#pragma unroll
  for (int k = 0; k < 4; ++k) cm[k] = s.colmax[(size_t)u * D + lane + 32 * k] & 0x7FFFu;
#pragma unroll
  for (int j = 0; j < G; ++j) {
    int pe[4], mx = INT_MIN;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      qw[j][k] = st.q[((size_t)u * G + j) * D + lane + 32 * k];
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
  // channel list: T8-class first, then T12/T16 (ascending channel inside each class)
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t b8[4], bf[4], bm16[4];
  int n8 = 0, nf = 0, n16 = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    b8[k] = __ballot_sync(0xFFFFFFFFu, ucode[k] == 8);
    bf[k] = __ballot_sync(0xFFFFFFFFu, ucode[k] >= 12);
    bm16[k] = __ballot_sync(0xFFFFFFFFu, ucode[k] == 16);
    n8 += __popc(b8[k]);
    nf += __popc(bf[k]);
    n16 += __popc(bm16[k]);
  }
  const int nl = n8 + nf;
  const int nlp = (nl + 7) & ~7;
  int base8 = 0, basef = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int c = lane + 32 * k;
    int pos = -1;
    if (ucode[k] == 8) pos = base8 + __popc(b8[k] & lt);
    else if (ucode[k] >= 12) pos = n8 + basef + __popc(bf[k] & lt);
    if (pos >= 0) {
      ws.ent[pos] = (uint16_t)(c | (ucode[k] << 8));
#pragma unroll
      for (int j = 0; j < G; ++j) {
        reinterpret_cast<uint16_t*>(ws.q[j])[pos] = code[j][k] ? (uint16_t)qw[j][k] : (uint16_t)0;
        if (G > 1) {
          const int cd = code[j][k];
          ws.hm[j][pos] = cd >= 16 ? make_uint2(0xFFFFFFFFu, 0u)
                                   : (cd == 12 ? make_uint2(0xFFF0FFF0u, 0x00080008u) : make_uint2(0xFF00FF00u, 0x00800080u));
        }
      }
    }
    base8 += __popc(b8[k]);
    basef += __popc(bf[k]);
  }
  for (int pos = nl + lane; pos < nlp; pos += 32) {
    ws.ent[pos] = 0;
#pragma unroll
    for (int j = 0; j < G; ++j) reinterpret_cast<uint16_t*>(ws.q[j])[pos] = 0;
  }
  if (book && lane == 0) {
    st.unit_bytes[(size_t)u * 4 + 0] = (int64_t)n * nl + (int64_t)(n / 2) * (nf + n16);
    st.unit_bytes[(size_t)u * 4 + 1] = 0;
  }
  if (lane == 0) {
    ws.nlist = nlp;
    ws.unit = u;
  }
  __syncwarp();
}

template <int G, bool TRUNC>
__global__ void __launch_bounds__(128) qk_kernel(akv_store_t s, akv_cfg_t cfg, akv_step_t st, int cap,
                                                 float inv_sqrt_d, int npg_max) {
  __shared__ QkWarp<G> wsm[4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  QkWarp<G>& ws = wsm[warp];
  if (lane == 0) ws.unit = -1;
  __syncwarp();
  const uint64_t pol = evict_first_policy();
  const unsigned total = (unsigned)s.n_units * npg_max;
  uint32_t tkm = 0xFFFFFFFFu, tf = 0u;
  if (TRUNC) {
    const int kb = cfg.trunc_bits - 6;
    const uint32_t km = (0xFFFFu << (10 - kb)) & 0xFFFFu;
    const uint32_t fill = kb < 10 ? (1u << (9 - kb)) : 0u;
    tkm = km | (km << 16);
    tf = fill | (fill << 16);
  }

  for (;;) {
    unsigned item = 0;
    if (lane == 0) item = atomicAdd(st.work + 0, 1u);
    item = __shfl_sync(0xFFFFFFFFu, item, 0);
    if (item >= total) break;
    const int u = item / npg_max, pg = item % npg_max;
    const int n = s.lengths[u];
    if (pg * P >= n) continue;
    if (ws.unit != u || pg == 0) k_prologue<G, TRUNC>(ws, s, cfg, st, u, n, pg == 0);

    const uint8_t* base = page_ptr(s.k_pool, s.page_table, s.max_pages, u, pg);
    const uint8_t* hb = base + lane * 8;
    const uint8_t* mb = base + MID + lane * 4;
    float acc[G][8];
#pragma unroll
    for (int j = 0; j < G; ++j)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[j][e] = 0.f;

    const int nb = ws.nlist >> 3;
    KBatch A, B;
    if (nb > 0) k_load<G>(A, ws, 0, hb, mb, pol);
    for (int b = 0; b < nb; b += 2) {
      if (b + 1 < nb) k_load<G>(B, ws, b + 1, hb, mb, pol);
      k_compute<G, TRUNC>(A, ws, b, acc, tkm, tf);
      if (b + 1 >= nb) break;
      if (b + 2 < nb) k_load<G>(A, ws, b + 2, hb, mb, pol);
      k_compute<G, TRUNC>(B, ws, b + 1, acc, tkm, tf);
    }

    // epilogue: scores + page softmax stats
    const int tok0 = pg * P + lane * 8;
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
  // self-resetting queue: the last warp out rewinds it for the next launch
  if (lane == 0) {
    __threadfence();
    const unsigned done = atomicAdd(st.work + 1, 1u);
    if (done == gridDim.x * 4 - 1) {
      st.work[0] = 0;
      st.work[1] = 0;
      __threadfence();
    }
  }
}

template <typename K>
int resident_blocks(K kernel, size_t smem = 0) {
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, 128, smem);
  return max(1, sms * max(per, 1));
}

template <int G, bool TRUNC>
static void launch_qk_t(const akv_store_t& s, const akv_cfg_t& cfg, const akv_step_t& st, int max_len,
                        cudaStream_t stream) {
  static int resident = 0;
  if (!resident) resident = resident_blocks(qk_kernel<G, TRUNC>);
  const int cap = s.max_pages * P;
  const int npg = (max_len + P - 1) / P;
  const long long items = (long long)s.n_units * npg;
  const int grid = (int)std::min<long long>(resident, (items + 3) / 4);
  const float isd = (float)(1.0 / 11.313708498984761);  // 1/sqrt(128)
  qk_kernel<G, TRUNC><<<max(grid, 1), 128, 0, stream>>>(s, cfg, st, cap, isd, npg);
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
