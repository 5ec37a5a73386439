// scores_aligned for every (unit, q-head) of a batch.
//
// Warp-specialised persistent kernel, one CTA per SM, 6-stage shared ring of
// half pages (64 channels x 256 tokens: 16 KB head plane + up to 8 KB mid +
// 8 KB low rows), two half-page stages per page:
//
//  producer warp   walks a contiguous range of (unit, page) items, evaluates
//                  Rule 1 for the unit's q-heads once per unit (rule1_target
//                  SPEC.md:157-165, required_mantissa_bits :139-147,
//                  tier_for_bits :148-156, k_channel_tiers :175-183, SURVEY
//                  App. A A-K/D1/D2/D8; the next unit's q and ColMax are
//                  prefetched), builds per half a channel list ordered by union
//                  class (T8 first, then T12/T16; SKIP channels dropped), and
//                  fills the stage: the 16 KB head-plane half by one TMA bulk
//                  copy (cp.async.bulk + mbarrier complete_tx) and only the
//                  128 B mid / low channel rows the union tier needs by
//                  cp.async from all 32 lanes (TMA pays a fixed cost per bulk
//                  copy, too high for 128 B rows);
//  8 consumer      warps (the channel list split over them) rebuild the fp16 words from
//                  shared memory with PRMT/LOP3 (midpoint fill for absent
//                  nibbles, HB:160-179) in two branch-free loops (T8 class,
//                  T12/T16 class) and accumulate q_c * K~ with the
//                  mixed-precision FHFMA (exact fp16 x fp16 products, fp32
//                  sums, D9); the 1/sqrt(d) scale is applied
//                  after accumulation; each page also yields its
//                  (max, sum exp) for the split softmax.
//
// Work split over the 8 consumer warps: the channel list is split 8/G ways per
// head and partial sums are reduced through shared memory in a fixed order;
// G = 8 gives every warp one head over all channels.  Each page's result is independent of which CTA
// or group computes it: the kernel is deterministic.
#include <algorithm>

#include "akv_common.cuh"

namespace akv {

#if AKV_PROBE == 3  // measurement aid: cycle accounting of the ring (tools/build_probe.sh)
__device__ unsigned long long qk_prof[16];
#define QK_T0(v) const long long v = clock64()
#define QK_ACC(var, t0) var += clock64() - (t0)
#else
#define QK_T0(v)
#define QK_ACC(var, t0)
#endif

constexpr int QK_NS = 6;                 // ring stages (half pages)
constexpr int QK_PRODUCERS = 2;          // producer warp h fills the half-page stages of half h
constexpr int QK_THREADS = 32 * (QK_PRODUCERS + 8);  // 2 producer + 8 consumer warps
constexpr int HCH = D / 2;               // channels per half page
constexpr int QS = HCH * P * 2;          // 32 KB stage: head [64][256] | mid [64][128] | low [64][128]
constexpr int QS_MID = HCH * P, QS_LOW = HCH * P + HCH * (P / 2);

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

// Per-stage (half page) metadata; list order: T8 class first, both ranges padded to 8.
template <int G>
struct alignas(16) QkMeta {
  int item, u, pg, n;
  int n8p, nlist, half, pad;
  uint16_t ent[HCH + 8];        // local channel (0..63) | has_low << 8 ; pads: channel 0, q = 0
  uint32_t q[G][HCH / 2 + 4];   // q (fp16) per list position, pairs; 0 for SKIP heads / pads
  uint8_t code[G][HCH + 8];     // per-head read code per list position (8/12/16; SKIP -> 8 with q = 0)
};

template <int G>
struct QkSplit {
  static constexpr int CS = G >= 8 ? 1 : 8 / G;  // ways the channel list is split over the 8 consumer warps
  static constexpr int HW = G >= 8 ? G / 8 : 1;  // heads per consumer warp
  static constexpr int NRED = CS > 1 ? 2 : 1;    // double-buffered partial sums (one barrier per page)
};

template <int G>
struct alignas(128) QkSmem {
  uint8_t data[QK_NS][QS];
  QkMeta<G> meta[QK_NS];
  QkMeta<G> cache[2];                    // producer-private: the current unit's lists (one per half)
  float red[QkSplit<G>::NRED][8][P];     // partial token sums per consumer warp (channel split)
  uint64_t full[QK_NS], empty[QK_NS];
};

__device__ __forceinline__ uint32_t ent_of(const uint4& e, int i) {
  const uint32_t w = i < 2 ? e.x : (i < 4 ? e.y : (i < 6 ? e.z : e.w));
  return (i & 1) ? (w >> 16) : (w & 0xFFFFu);
}

// ----------------------------------------------------------------------------
// producer
// ----------------------------------------------------------------------------
template <int G>
struct QkUnit {
  UnitPages pages;
  uint32_t cm[4];
  uint32_t qw[G][4];
};

// Issue the loads a unit's Rule-1 prologue needs (no wait: consumed later).
template <int G>
__device__ __forceinline__ void qk_fetch_unit(QkUnit<G>& f, const akv_store_t& s, const akv_step_t& st, int u) {
  const int lane = threadIdx.x & 31;
  unit_pages_fetch(f.pages, s, u);
#pragma unroll
  for (int k = 0; k < 4; ++k) f.cm[k] = s.colmax[(size_t)u * D + lane + 32 * k];
#pragma unroll
  for (int j = 0; j < G; ++j)
#pragma unroll
    for (int k = 0; k < 4; ++k) f.qw[j][k] = st.q[((size_t)u * G + j) * D + lane + 32 * k];
}

// Rule 1 for one unit (all q-heads): tier codes, the two half lists and the
// fetch masks; once per unit per CTA.  `book`: this CTA owns the unit's page 0
// and writes the per-step bookkeeping (K tiers, K counters, status, bytes).
// Lane l owns channels l + 32k (k = 0..3): words k = 0, 1 are half 0.
template <int G, bool TRUNC>
__device__ void qk_unit_prologue(QkSmem<G>& sm, const QkUnit<G>& f, bool book, int my_hf, const akv_cfg_t& cfg,
                                 const akv_step_t& st, uint32_t (&bm)[4], uint32_t (&bl)[4]) {
  const int lane = threadIdx.x & 31;
  const bool aligned = cfg.force_tier == 0 && !TRUNC;
  int code[G][4], ucode[4] = {0, 0, 0, 0};
#pragma unroll
  for (int j = 0; j < G; ++j) {
    int pe[4], mx = INT_MIN;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t qw = f.qw[j][k];
      const uint32_t cmk = f.cm[k] & 0x7FFFu;
      const bool valid = (qw & 0x7FFFu) && cmk && finite16(qw);
      pe[k] = valid ? magexp16(qw) + magexp16(cmk) + 1 : INT_MIN;
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
        const bool qz = (f.qw[j][k] & 0x7FFFu) == 0, cz = (f.cm[k] & 0x7FFFu) == 0;
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
    if (book) {  // per-step bookkeeping, once per unit
      const size_t h = (size_t)f.pages.u * G + j;
      int c8 = 0, c12 = 0, c16 = 0, bad = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        st.k_tiers[h * D + lane + 32 * k] = (uint8_t)code[j][k];
        c8 += __popc(__ballot_sync(0xFFFFFFFFu, code[j][k] == 8));
        c12 += __popc(__ballot_sync(0xFFFFFFFFu, code[j][k] == 12));
        c16 += __popc(__ballot_sync(0xFFFFFFFFu, code[j][k] == 16));
        bad += __popc(__ballot_sync(0xFFFFFFFFu, !finite16(f.qw[j][k])));
      }
      if (lane == 0) {
        int64_t* ct = st.counters + h * 8;
        ct[0] = (int64_t)c8 * f.pages.n;
        ct[1] = (int64_t)c12 * f.pages.n;
        ct[2] = (int64_t)c16 * f.pages.n;
        ct[3] = ct[4] = ct[5] = ct[6] = ct[7] = 0;
        long long w = 0;
        if (bad) w = status_word(AKV_STATUS_BAD_Q, 0);
        else if (aligned && maxpe == INT_MIN) w = status_word(AKV_STATUS_DEGENERATE, 0);
        st.status[h] = w;
      }
    }
  }
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t b8[4];
  int nh = 0, nm_all = 0, nl_all = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    b8[k] = __ballot_sync(0xFFFFFFFFu, ucode[k] == 8);
    bm[k] = __ballot_sync(0xFFFFFFFFu, ucode[k] >= 12);
    bl[k] = __ballot_sync(0xFFFFFFFFu, ucode[k] == 16);
    nh += __popc(b8[k]) + __popc(bm[k]);
    nm_all += __popc(bm[k]);
    nl_all += __popc(bl[k]);
  }
#pragma unroll
  for (int hf = 0; hf < 2; ++hf) {
    if (hf != my_hf) continue;  // each producer builds only its own half's list
    QkMeta<G>& mt = sm.cache[hf];
    const int n8 = __popc(b8[2 * hf]) + __popc(b8[2 * hf + 1]);
    const int nm = __popc(bm[2 * hf]) + __popc(bm[2 * hf + 1]);
    const int n8p = (n8 + 7) & ~7, nlp = n8p + ((nm + 7) & ~7);
    int base8 = 0, basem = 0;
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      const int k = 2 * hf + kk;
      const int cl = lane + 32 * kk;  // channel inside the half
      int pos = -1;
      if (ucode[k] == 8) pos = base8 + __popc(b8[k] & lt);
      else if (ucode[k] >= 12) pos = n8p + basem + __popc(bm[k] & lt);
      if (pos >= 0) {
        mt.ent[pos] = (uint16_t)(cl | ((ucode[k] == 16 ? 1 : 0) << 8));
#pragma unroll
        for (int j = 0; j < G; ++j) {
          reinterpret_cast<uint16_t*>(mt.q[j])[pos] = code[j][k] ? (uint16_t)f.qw[j][k] : (uint16_t)0;
          mt.code[j][pos] = (uint8_t)(code[j][k] ? code[j][k] : 8);
        }
      }
      base8 += __popc(b8[k]);
      basem += __popc(bm[k]);
    }
    // pads (channel 0, q = 0): the head plane is always resident, so the word is finite and adds 0
    if (lane < 8) {
      const int p0 = n8 + lane, p1 = n8p + nm + lane;
      if (p0 < n8p) {
        mt.ent[p0] = 0;
#pragma unroll
        for (int j = 0; j < G; ++j) {
          reinterpret_cast<uint16_t*>(mt.q[j])[p0] = 0;
          mt.code[j][p0] = 8;
        }
      }
      if (p1 < nlp) {
        mt.ent[p1] = 0;
#pragma unroll
        for (int j = 0; j < G; ++j) {
          reinterpret_cast<uint16_t*>(mt.q[j])[p1] = 0;
          mt.code[j][p1] = 8;
        }
      }
    }
    if (lane == 0) {
      mt.n8p = n8p;
      mt.nlist = nlp;
      mt.half = hf;
    }
  }
  if (book && lane == 0) {
    st.unit_bytes[(size_t)f.pages.u * 4 + 0] = (int64_t)f.pages.n * nh + (int64_t)(f.pages.n / 2) * (nm_all + nl_all);
    st.unit_bytes[(size_t)f.pages.u * 4 + 1] = 0;
  }
  __syncwarp();
}

// Publish one half page into a ring stage: the cached half list + item fields,
// then the copies (head half by TMA bulk copy; needed mid / low rows by cp.async).
template <int G>
__device__ void qk_stage(QkSmem<G>& sm, int stage, int hf, int item, int u, int pg, int n, const uint8_t* src,
                         const uint32_t (&bm)[4], const uint32_t (&bl)[4]) {
  const int lane = threadIdx.x & 31;
  QK_T0(t_a);
  QkMeta<G>& mt = sm.meta[stage];
  constexpr int W = sizeof(QkMeta<G>) / 16;
  const uint4* srcm = reinterpret_cast<const uint4*>(&sm.cache[hf]);
  uint4* dstm = reinterpret_cast<uint4*>(&mt);
  for (int i = lane; i < W; i += 32) dstm[i] = srcm[i];
  __syncwarp();
  if (lane == 0) {
    mt.item = item;
    mt.u = u;
    mt.pg = pg;
    mt.n = n;
  }
  uint8_t* dst = sm.data[stage];
  __syncwarp();
#if AKV_PROBE == 3
  long long t_b = clock64();
  if (lane == 0) atomicAdd(&qk_prof[11], (unsigned long long)(t_b - t_a));
#endif
#if AKV_PROBE == 2  // measurement aid: no plane loads (consumer-bound time)
  if (lane == 0) mbar_arrive(&sm.full[stage]);
#else
  if (lane == 0) {
    mbar_arrive_expect_tx(&sm.full[stage], HCH * P);
    bulk_g2s(dst, src + hf * HCH * P, HCH * P, &sm.full[stage]);
  }
#if AKV_PROBE == 3
  __syncwarp();
  long long t_c = clock64();
  if (lane == 0) atomicAdd(&qk_prof[8], (unsigned long long)(t_c - t_b));
#endif
  const uint32_t mm[2] = {hf ? bm[2] : bm[0], hf ? bm[3] : bm[1]};
  const uint32_t ml[2] = {hf ? bl[2] : bl[0], hf ? bl[3] : bl[1]};
  cp_rows<2, P / 2>(mm, dst + QS_MID, src + MID + hf * HCH * (P / 2));
  cp_rows<2, P / 2>(ml, dst + QS_LOW, src + LOW + hf * HCH * (P / 2));
#endif
#if AKV_PROBE == 3
  __syncwarp();
  long long t_d = clock64();
  if (lane == 0) atomicAdd(&qk_prof[9], (unsigned long long)(t_d - t_c));
#endif
  cp_async_arrive_noinc(&sm.full[stage]);
#if AKV_PROBE == 3
  __syncwarp();
  if (lane == 0) atomicAdd(&qk_prof[10], (unsigned long long)(clock64() - t_d));
#endif
}

// ----------------------------------------------------------------------------
// consumer
// ----------------------------------------------------------------------------
template <int G, bool TRUNC>
__device__ __forceinline__ void qk_consume_half(const QkSmem<G>& sm, int stage, int w8, float (&acc)[QkSplit<G>::HW][8],
                                                uint32_t tkm, uint32_t tf) {
  constexpr int CS = QkSplit<G>::CS, HW = QkSplit<G>::HW;
  const int lane = threadIdx.x & 31;
  const QkMeta<G>& mt = sm.meta[stage];
  const uint8_t* pgd = sm.data[stage];
  const int cs = w8 % CS;
  const int j0 = (w8 / CS) * HW;
  const int nb8 = mt.n8p >> 3, nb = mt.nlist >> 3;
  const uint8_t* hb = pgd + lane * 8;
  const uint8_t* mb = pgd + QS_MID + lane * 4;

  // T8-class channels: head byte only (every q-head reads T8, or SKIP with q = 0)
  for (int b = cs; b < nb8; b += CS) {
    const uint4 e4 = *reinterpret_cast<const uint4*>(&mt.ent[b * 8]);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t ch = ent_of(e4, i) & 0xFFu;
      const uint2 h = *reinterpret_cast<const uint2*>(hb + ch * P);
      const uint32_t c80 = 0x80808080u;
      uint32_t w[4];
      w[0] = prmt(h.x, c80, 0x1404);
      w[1] = prmt(h.x, c80, 0x3424);
      w[2] = prmt(h.y, c80, 0x1404);
      w[3] = prmt(h.y, c80, 0x3424);
      if (TRUNC) {
#pragma unroll
        for (int k = 0; k < 4; ++k) w[k] = (w[k] & tkm) | tf;
      }
#pragma unroll
      for (int jj = 0; jj < HW; ++jj) {
        const uint32_t qp = mt.q[j0 + jj][b * 4 + (i >> 1)];
        if (i & 1) fma8<1>(w, qp, acc[jj]);
        else fma8<0>(w, qp, acc[jj]);
      }
    }
  }
  // T12/T16-class channels: head + mid (+ low) rows
  const int bf0 = nb8 + ((cs - nb8 % CS) % CS + CS) % CS;
  for (int b = bf0; b < nb; b += CS) {
    const uint4 e4 = *reinterpret_cast<const uint4*>(&mt.ent[b * 8]);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t en = ent_of(e4, i);
      const uint32_t ch = en & 0xFFu;
      const uint2 h = *reinterpret_cast<const uint2*>(hb + ch * P);
      const uint32_t m = *reinterpret_cast<const uint32_t*>(mb + ch * (P / 2));
      uint32_t l = 0x88888888u;
      if (en >> 8) l = *reinterpret_cast<const uint32_t*>(mb + (QS_LOW - QS_MID) + ch * (P / 2));
      uint32_t w[4];
      assemble8(h.x, h.y, m, l, w);
      if (TRUNC) {
#pragma unroll
        for (int k = 0; k < 4; ++k) w[k] = (w[k] & tkm) | tf;
      }
#pragma unroll
      for (int jj = 0; jj < HW; ++jj) {
        const int j = j0 + jj;
        uint32_t wj[4];
        if (G > 1) {
          const uint32_t cd = mt.code[j][b * 8 + i];
          const uint32_t km = cd >= 16 ? 0xFFFFFFFFu : (cd == 12 ? 0xFFF0FFF0u : 0xFF00FF00u);
          const uint32_t fl = cd >= 16 ? 0u : (cd == 12 ? 0x00080008u : 0x00800080u);
#pragma unroll
          for (int k = 0; k < 4; ++k) wj[k] = (w[k] & km) | fl;
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k) wj[k] = w[k];
        }
        const uint32_t qp = mt.q[j][b * 4 + (i >> 1)];
        if (i & 1) fma8<1>(wj, qp, acc[jj]);
        else fma8<0>(wj, qp, acc[jj]);
      }
    }
  }
}

// Scale, store and summarise the scores of T consecutive tokens per lane
// (tokens tok0 .. tok0+T-1, tok0 = first token of this lane): per 32-token
// chunk (32/T lanes) the (max, sum exp) pair for the split softmax.
template <int T>
__device__ __forceinline__ void qk_finish(const float (&raw)[T], int tok0, int n, float* scores_h, float* stats_h,
                                          float isd) {
  constexpr int LPC = 32 / T;  // lanes per 32-token chunk
  const int lane = threadIdx.x & 31;
  const int nv = min(max(n - tok0, 0), T);
  float sv[T];
  float m = -INFINITY;
#pragma unroll
  for (int e = 0; e < T; ++e) {
    sv[e] = raw[e] * isd;
    if (e < nv) m = fmaxf(m, sv[e]);
  }
#pragma unroll
  for (int o = 1; o < LPC; o <<= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
  float l = 0.f;
#pragma unroll
  for (int e = 0; e < T; ++e)
    if (e < nv) l += expf(sv[e] - m);
#pragma unroll
  for (int o = 1; o < LPC; o <<= 1) l += __shfl_xor_sync(0xFFFFFFFFu, l, o);
  float* out = scores_h + tok0;
  if (nv == T) {
    if constexpr (T == 1) {
      out[0] = sv[0];
    } else if constexpr (T == 2) {
      *reinterpret_cast<float2*>(out) = make_float2(sv[0], sv[1]);
    } else {
#pragma unroll
      for (int e = 0; e < T; e += 4) *reinterpret_cast<float4*>(out + e) = make_float4(sv[e], sv[e + 1], sv[e + 2], sv[e + 3]);
    }
  } else {
#pragma unroll
    for (int e = 0; e < T; ++e)
      if (e < nv) out[e] = sv[e];
  }
  if (lane % LPC == 0 && tok0 < n) {
    float* ps = stats_h + (tok0 >> 5) * 2;
    ps[0] = m;
    ps[1] = l;
  }
}

template <int G, bool TRUNC>
__global__ void __launch_bounds__(QK_THREADS, 1) qk_kernel(akv_store_t s, akv_cfg_t cfg, akv_step_t st, int cap,
                                                           float isd, int npg_max) {
  constexpr int CS = QkSplit<G>::CS, HW = QkSplit<G>::HW;
  extern __shared__ __align__(128) uint8_t qk_smem_raw[];
  QkSmem<G>& sm = *reinterpret_cast<QkSmem<G>*>(qk_smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < QK_NS; ++i) {
      mbar_init(&sm.full[i], 33);  // expect_tx arrival + 32 cp.async arrivals
      mbar_init(&sm.empty[i], 8);  // one arrival per consumer warp
    }
    mbar_fence_init();
  }
  __syncthreads();
  const long long total = (long long)s.n_units * npg_max;

  if (warp < QK_PRODUCERS) {
    // ---------------- producers: contiguous item range, Rule 1 once per unit ----------------
    // Both producers walk the same items; producer h fills the stages of half h.
    const int my_hf = warp;
    const long long per = (total + gridDim.x - 1) / gridDim.x;
    const long long i0 = (long long)blockIdx.x * per, i1 = min(total, i0 + per);
#if AKV_PROBE == 3
    long long p_wait = 0, p_issue = 0;
    const long long p_start = clock64();
#endif
    QkUnit<G> cur, nxt;
    uint32_t bm[4] = {0, 0, 0, 0}, bl[4] = {0, 0, 0, 0};
    int cur_u = -1;
    if (i0 < i1) qk_fetch_unit<G>(nxt, s, st, (int)(i0 / npg_max));
    int k = 0;
    for (long long idx = i0; idx < i1; ++idx) {
      const int u = (int)(idx / npg_max), pg = (int)(idx % npg_max);
      if (u != cur_u) {
        cur = nxt;
        if ((long long)(u + 1) * npg_max < i1) qk_fetch_unit<G>(nxt, s, st, u + 1);  // prefetch the next unit
        cur_u = u;
        if (cur.pages.n > 0) qk_unit_prologue<G, TRUNC>(sm, cur, pg == 0 && my_hf == 0, my_hf, cfg, st, bm, bl);
      }
      if (pg * P >= cur.pages.n) continue;  // beyond this unit's length (ragged batch)
      const uint8_t* src = s.k_pool + unit_page(cur.pages, s, pg) * PAGE;
      {
        const int kk = k + my_hf, stage = kk % QK_NS;
        QK_T0(tw);
        mbar_wait(&sm.empty[stage], ((kk / QK_NS) & 1) ^ 1);
        QK_ACC(p_wait, tw);
        QK_T0(ti);
        qk_stage<G>(sm, stage, my_hf, (int)idx, u, pg, cur.pages.n, src, bm, bl);
        QK_ACC(p_issue, ti);
        k += 2;
      }
    }
#if AKV_PROBE == 3
    if (lane == 0) {
      atomicAdd(&qk_prof[0], (unsigned long long)p_wait);
      atomicAdd(&qk_prof[1], (unsigned long long)p_issue);
      atomicAdd(&qk_prof[2], (unsigned long long)(clock64() - p_start));
    }
#endif
    // terminator: this producer's half of the next page slot
    {
      const int kk = k + my_hf, stage = kk % QK_NS;
      mbar_wait(&sm.empty[stage], ((kk / QK_NS) & 1) ^ 1);
      if (lane == 0) sm.meta[stage].item = -1;
      __syncwarp();
      mbar_arrive(&sm.full[stage]);                 // 32 lane arrivals ...
      if (lane == 0) mbar_arrive(&sm.full[stage]);  // ... + the expect_tx slot
      __syncwarp();
    }
  } else {
    // ---------------- consumers: eight warps share each page ----------------
    const int w8 = warp - QK_PRODUCERS;
    uint32_t tkm = 0xFFFFFFFFu, tf = 0u;
    if (TRUNC) {
      const int kb = cfg.trunc_bits - 6;
      const uint32_t km = (0xFFFFu << (10 - kb)) & 0xFFFFu;
      const uint32_t fill = kb < 10 ? (1u << (9 - kb)) : 0u;
      tkm = km | (km << 16);
      tf = fill | (fill << 16);
    }
    const int cs = w8 % CS, j0 = (w8 / CS) * HW;
#if AKV_PROBE == 3
    long long c_wait = 0, c_comp = 0;
    const long long c_start = clock64();
#endif
    for (int kp = 0;; ++kp) {
      float acc[HW][8];
#pragma unroll
      for (int jj = 0; jj < HW; ++jj)
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[jj][e] = 0.f;
      int u = 0, pg = 0, n = 0;
      bool done = false;
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        const int kk = 2 * kp + hf, stage = kk % QK_NS;
        QK_T0(cw);
        mbar_wait(&sm.full[stage], (kk / QK_NS) & 1);
        QK_ACC(c_wait, cw);
        if (sm.meta[stage].item < 0) {
          done = true;
          break;
        }
        if (hf == 0) {
          u = sm.meta[stage].u;
          pg = sm.meta[stage].pg;
          n = sm.meta[stage].n;
        }
#if AKV_PROBE != 1  // measurement aid: 1 = no consumer compute (load-bound time)
        QK_T0(cc);
        qk_consume_half<G, TRUNC>(sm, stage, w8, acc, tkm, tf);
        QK_ACC(c_comp, cc);
#endif
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[stage]);  // stage no longer read by this warp
      }
      if (done) {
#if AKV_PROBE == 3
        if (lane == 0) {
          atomicAdd(&qk_prof[3], (unsigned long long)c_wait);
          atomicAdd(&qk_prof[4], (unsigned long long)c_comp);
          atomicAdd(&qk_prof[5], (unsigned long long)(clock64() - c_start));
          
        }
#endif
        break;
      }
      const int cap_chunks = s.max_pages * (P / 32);
      if constexpr (CS == 1) {
#pragma unroll
        for (int jj = 0; jj < HW; ++jj) {
          const size_t hh = (size_t)u * G + j0 + jj;
          qk_finish<8>(acc[jj], pg * P + lane * 8, n, st.scores + hh * cap, st.page_stats + hh * cap_chunks * 2, isd);
        }
      } else {
        // channel split: the CS warps of a head publish their partial sums, then each
        // reduces its own 256/CS-token slice in a fixed order (deterministic).  The
        // double buffer makes one barrier per page enough.
        float* rw = sm.red[kp & 1][w8];
        *reinterpret_cast<float4*>(rw + lane * 8) = make_float4(acc[0][0], acc[0][1], acc[0][2], acc[0][3]);
        *reinterpret_cast<float4*>(rw + lane * 8 + 4) = make_float4(acc[0][4], acc[0][5], acc[0][6], acc[0][7]);
        named_bar(1, 256);
        constexpr int T = G;  // tokens per lane in the reduction: 256 / CS / 32
        const int tk = cs * (P / CS) + lane * T;
        float sum[T];
#pragma unroll
        for (int e = 0; e < T; ++e) sum[e] = 0.f;
#pragma unroll
        for (int c2 = 0; c2 < CS; ++c2) {
          const float* r2 = sm.red[kp & 1][w8 - cs + c2] + tk;
          if constexpr (T == 1) {
            sum[0] += r2[0];
          } else if constexpr (T == 2) {
            const float2 a = *reinterpret_cast<const float2*>(r2);
            sum[0] += a.x;
            sum[1] += a.y;
          } else {
            const float4 a = *reinterpret_cast<const float4*>(r2);
            sum[0] += a.x;
            sum[1] += a.y;
            sum[2] += a.z;
            sum[3] += a.w;
          }
        }
        const size_t hh = (size_t)u * G + j0;
        qk_finish<T>(sum, pg * P + tk, n, st.scores + hh * cap, st.page_stats + hh * cap_chunks * 2, isd);
      }
    }
  }
}

template <int G>
constexpr bool qk_smem_fits = sizeof(QkSmem<G>) <= 232448;
static_assert(qk_smem_fits<1> && qk_smem_fits<2> && qk_smem_fits<4> && qk_smem_fits<8>, "QK shared memory > 227 KB");

template <int G, bool TRUNC>
static void launch_qk_t(const akv_store_t& s, const akv_cfg_t& cfg, const akv_step_t& st, int max_len,
                        cudaStream_t stream) {
  static int sms = 0;
  const size_t smem = sizeof(QkSmem<G>);
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(qk_kernel<G, TRUNC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  const int cap = s.max_pages * P;
  const int npg = (max_len + P - 1) / P;
  const long long items = (long long)s.n_units * npg;
  const int grid = (int)std::min<long long>(sms, std::max<long long>(items / 2, 1));
  const float isd = (float)(1.0 / 11.313708498984761);  // 1/sqrt(128)
  qk_kernel<G, TRUNC><<<grid, QK_THREADS, smem, stream>>>(s, cfg, st, cap, isd, npg);
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

#if AKV_PROBE == 3
extern "C" int akv_probe_read_qk(unsigned long long* host) {
  cudaMemcpyFromSymbol(host, akv::qk_prof, sizeof(akv::qk_prof));
  unsigned long long z[16] = {};
  cudaMemcpyToSymbol(akv::qk_prof, z, sizeof(z));
  return 0;
}
#endif
