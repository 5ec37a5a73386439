// output_aligned for every (unit, q-head): persistent warps
// pull (unit, page) items from an atomic queue; one item = one 256-token V
// page; the page's partial output goes to o_partial[h][page] and the combine
// kernel adds o_est and the partials in a fixed order (deterministic).
//
// Per item prologue (one lane per row) decides, for every row t and q-head j,
// a mode:
//   SKIP     t was selected by the estimate (D6: its T16 contribution is in
//            o_est) or t >= n;
//   T8       p_t == 0 (D5), or the RowMax superset bound shows every element of
//            the row needs <= 2 kept bits (H6: e_v <= max(bexp(RowMax_t),1)-15,
//            target_r >= min_r target_r);
//   T8/T12/T16 forced tiers (D8), the row strategy (D7), baseline truncation;
//   ELEMENT  per-element rule from the head byte's exponent (D4): keep mid iff
//            max(bexp,1) + e(p_t) > 17 + target_r - margin, low iff > that + 4.
// The union over the kv-head's q-heads decides which 64 B nibble rows are
// fetched; per-element truncation is applied after the fetch, so the masks
// are exactly the oracle's.
//
// Main loop: 16 lanes per row x 8 channels per lane (LDG.64 head, LDG.32
// mid/low), two rows per warp instruction, loads software-pipelined one
// 16-row block ahead.  Blocks whose rows are all T8/SKIP take a branch-free
// path (4 PRMT per 8 elements).  fp16 -> fp32 by HADD2.F32, p_t * V~ by the
// packed FFMA2 into fp32 accumulators (>= 24-bit).
#include <algorithm>

#include "akv_common.cuh"

namespace akv {

enum : uint32_t { M_SKIP = 0, M_ELEM = 1, M_T8 = 8, M_T12 = 12, M_T16 = 16 };

template <int G>
struct alignas(16) PvWarp {
  float2 row[G][P];  // (p_t, bits(ep << 8 | mode)) per (head, row)
  int gthr[G][D];    // ELEMENT thresholds per (head, channel)
  uint8_t fl[P];     // union fetch flags: 2 = mid row, 4 = low row
  uint32_t blk_slow;
};

struct VBatch {
  uint2 h[8];
  uint32_t m[8], l[8];
};

template <int G>
__device__ __forceinline__ void v_load(VBatch& X, const PvWarp<G>& ws, int blk, int half, const uint8_t* hb,
                                       const uint8_t* mb, uint64_t pol) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = blk * 16 + 2 * i + half;
    const uint32_t f = ws.fl[r];
    X.h[i] = ld_stream_u64(hb + (blk * 16 + 2 * i) * D, pol);
    if (f & 2) X.m[i] = ld_stream_u32(mb + (blk * 16 + 2 * i) * (D / 2), pol);
    if (f & 4) X.l[i] = ld_stream_u32(mb + (blk * 16 + 2 * i) * (D / 2) + (LOW - MID), pol);
  }
}

__device__ __forceinline__ void t8_words(uint2 h, uint32_t w[4]) {
  const uint32_t c80 = 0x80808080u;
  w[0] = prmt(h.x, c80, 0x1404);
  w[1] = prmt(h.x, c80, 0x3424);
  w[2] = prmt(h.y, c80, 0x1404);
  w[3] = prmt(h.y, c80, 0x3424);
}

template <int G, bool TRUNC, bool EXPORT>
__device__ __forceinline__ void v_compute(const VBatch& X, const PvWarp<G>& ws, int blk, int half, int cl,
                                          float2 acc[G][4], int cnt[G][3], uint32_t tkm, uint32_t tf,
                                          uint8_t* vt_row0, size_t vt_head_stride, int rows_valid) {
  const bool slow = (ws.blk_slow >> blk) & 1u;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = blk * 16 + 2 * i + half;
    if (!slow) {
      // every row of the block is T8 or SKIP (p = 0) for every head
      uint32_t w[4];
      t8_words(X.h[i], w);
      float2 f[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) f[k] = half2_bits_to_float2(w[k]);
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const float p = ws.row[j][r].x;
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[j][k] = ffma2_scalar(f[k], p, acc[j][k]);
        if (EXPORT && vt_row0 && r < rows_valid) {
          const uint32_t mode = __float_as_uint(ws.row[j][r].y) & 0xFFu;
          const uint32_t c = mode == M_SKIP ? 0x10101010u : 0x08080808u;
          *reinterpret_cast<uint2*>(vt_row0 + j * vt_head_stride + (size_t)r * D + cl * 8) = make_uint2(c, c);
        }
      }
      continue;
    }
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const float2 rw = ws.row[j][r];
      const uint32_t em = __float_as_uint(rw.y);
      const uint32_t mode = em & 0xFFu;
      uint32_t w[4];
      uint32_t code_lo = 0, code_hi = 0;
      if (mode != M_ELEM) {
        const TierMask tm = tier_mask(mode == M_SKIP ? 8 : (int)mode);
        assemble8(X.h[i].x, X.h[i].y, bsel(tm.mk, X.m[i], 0x88888888u), bsel(tm.lk, X.l[i], tm.lf), w);
        if (EXPORT) code_lo = code_hi = (mode == M_SKIP ? 16u : mode) * 0x01010101u;
      } else {
        assemble8(X.h[i].x, X.h[i].y, X.m[i], X.l[i], w);
        const int ep = (int)em >> 8;
        const int4 g0 = *reinterpret_cast<const int4*>(&ws.gthr[j][cl * 8]);
        const int4 g1 = *reinterpret_cast<const int4*>(&ws.gthr[j][cl * 8 + 4]);
        const int gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const uint32_t hbyte = ((e < 4 ? X.h[i].x : X.h[i].y) >> (8 * (e & 3))) & 0xFFu;
          const int E = max((int)((hbyte >> 2) & 31u), 1) + ep;
          const bool km = E > gg[e], kl = E > gg[e] + 4;
          const int sh = 16 * (e & 1);
          uint32_t w16 = (w[e >> 1] >> sh) & 0xFFFFu;
          w16 = kl ? w16 : (km ? ((w16 & 0xFFF0u) | 0x8u) : ((w16 & 0xFF00u) | 0x80u));
          w[e >> 1] = (w[e >> 1] & ~(0xFFFFu << sh)) | (w16 << sh);
          cnt[j][kl ? 2 : (km ? 1 : 0)] += 1;
          if (EXPORT) {
            const uint32_t cd = kl ? 16u : (km ? 12u : 8u);
            if (e < 4) code_lo |= cd << (8 * e);
            else code_hi |= cd << (8 * (e - 4));
          }
        }
      }
      if (TRUNC) {
#pragma unroll
        for (int k = 0; k < 4; ++k) w[k] = (w[k] & tkm) | tf;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[j][k] = ffma2_scalar(half2_bits_to_float2(w[k]), rw.x, acc[j][k]);
      if (EXPORT && vt_row0 && r < rows_valid)
        *reinterpret_cast<uint2*>(vt_row0 + j * vt_head_stride + (size_t)r * D + cl * 8) = make_uint2(code_lo, code_hi);
    }
  }
}

template <int G, bool TRUNC, bool EXPORT>
__global__ void __launch_bounds__(128) pv_kernel(akv_store_t s, akv_cfg_t cfg, akv_step_t st, int cap, int npg_max) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  PvWarp<G>& ws = reinterpret_cast<PvWarp<G>*>(smem_raw)[warp];
  const uint64_t pol = evict_first_policy();
  const unsigned total = (unsigned)s.n_units * npg_max;
  const bool aligned = cfg.force_tier == 0 && !TRUNC;
  const uint32_t uniform = TRUNC ? 16u : (uint32_t)cfg.force_tier;
  const int half = lane >> 4, cl = lane & 15;
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
    if (lane == 0) item = atomicAdd(st.work + 2, 1u);
    item = __shfl_sync(0xFFFFFFFFu, item, 0);
    if (item >= total) break;
    const int u = item / npg_max, pg = item % npg_max;
    const int n = s.lengths[u];
    if (pg * P >= n) continue;
    const int rows_valid = min(n - pg * P, P);

    // ---------------- prologue: modes per (head, row) ----------------
    int cnt[G][3];
    int min_t[G], unk[G];
#pragma unroll
    for (int j = 0; j < G; ++j) {
      cnt[j][0] = cnt[j][1] = cnt[j][2] = 0;
      const int32_t* hm = st.head_meta + ((size_t)u * G + j) * 4;
      min_t[j] = hm[1];
      unk[j] = hm[2];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int tg = st.targets[((size_t)u * G + j) * D + lane + 32 * k];
        ws.gthr[j][lane + 32 * k] = tg == AKV_TARGET_UNKNOWN ? -(1 << 20) : 17 + tg - cfg.margin_bits;
      }
    }
    long long vbytes = 0;
    uint32_t blk_slow = 0;
#pragma unroll 1
    for (int k = 0; k < 8; ++k) {
      const int r = lane + 32 * k;
      const int t = pg * P + r;
      uint32_t fl = 0;
      bool nont8 = false;
      const uint32_t rm = t < n ? s.rowmax[(size_t)u * s.max_pages * P + t] : 0u;
      const int e_rm = max(bexp16(rm), 1) - 15;  // D4 bound on every element's e_v
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const size_t h = (size_t)u * G + j;
        uint32_t mode = M_SKIP;
        float p = 0.f;
        int ep = -30000;
        if (t < n) {
          p = st.probs[h * cap + t];
          if (p > 0.f) ep = floor_log2f(p);
          if (!aligned) {
            mode = uniform;
          } else if ((st.sel_bits[h * (cap >> 5) + (t >> 5)] >> (t & 31)) & 1u) {
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
              fl |= bound > 6 ? 6 : 2;
            } else {
              mode = M_T8;
            }
          }
        }
        if (mode == M_T12) fl |= 2;
        if (mode == M_T16) fl |= 6;
        if (mode == M_T8) cnt[j][0] += D;
        if (mode == M_T12) cnt[j][1] += D;
        if (mode == M_T16) cnt[j][2] += D;
        nont8 |= mode != M_SKIP && mode != M_T8;
        ws.row[j][r] = make_float2(p, __uint_as_float(((uint32_t)ep << 8) | mode));
      }
      ws.fl[r] = (uint8_t)fl;
      if (t < n) vbytes += D + ((fl & 2) ? D / 2 : 0) + ((fl & 4) ? D / 2 : 0);
      const uint32_t bs = __ballot_sync(0xFFFFFFFFu, nont8);
      blk_slow |= (((bs & 0xFFFFu) ? 1u : 0u) << (2 * k)) | (((bs >> 16) ? 1u : 0u) << (2 * k + 1));
    }
    if (lane == 0) ws.blk_slow = blk_slow;
    __syncwarp();

    // ---------------- main loop ----------------
    const uint8_t* base = page_ptr(s.v_pool, s.page_table, s.max_pages, u, pg);
    const uint8_t* hb = base + half * D + cl * 8;
    const uint8_t* mb = base + MID + half * (D / 2) + cl * 4;
    const int nblk = (rows_valid + 15) >> 4;
    float2 acc[G][4];
#pragma unroll
    for (int j = 0; j < G; ++j)
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[j][k] = make_float2(0.f, 0.f);
    uint8_t* vt0 = nullptr;
    size_t vstride = 0;
    if (EXPORT && st.v_tiers) {
      vt0 = st.v_tiers + ((size_t)u * G * cap + (size_t)pg * P) * D;
      vstride = (size_t)cap * D;
    }
    VBatch A, B;
    v_load<G>(A, ws, 0, half, hb, mb, pol);
    for (int b = 0; b < nblk; b += 2) {
      if (b + 1 < nblk) v_load<G>(B, ws, b + 1, half, hb, mb, pol);
      v_compute<G, TRUNC, EXPORT>(A, ws, b, half, cl, acc, cnt, tkm, tf, vt0, vstride, rows_valid);
      if (b + 1 >= nblk) break;
      if (b + 2 < nblk) v_load<G>(A, ws, b + 2, half, hb, mb, pol);
      v_compute<G, TRUNC, EXPORT>(B, ws, b + 1, half, cl, acc, cnt, tkm, tf, vt0, vstride, rows_valid);
    }

    // ---------------- epilogue: partial o of this page, counters ----------------
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const size_t h = (size_t)u * G + j;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        acc[j][k].x += __shfl_xor_sync(0xFFFFFFFFu, acc[j][k].x, 16);
        acc[j][k].y += __shfl_xor_sync(0xFFFFFFFFu, acc[j][k].y, 16);
      }
      if (half == 0) {
        float4* dst = reinterpret_cast<float4*>(st.o_partial + (h * s.max_pages + pg) * D + cl * 8);
        dst[0] = make_float4(acc[j][0].x, acc[j][0].y, acc[j][1].x, acc[j][1].y);
        dst[1] = make_float4(acc[j][2].x, acc[j][2].y, acc[j][3].x, acc[j][3].y);
      }
      const int a = warp_sum_i(cnt[j][0]), bq = warp_sum_i(cnt[j][1]), c = warp_sum_i(cnt[j][2]);
      if (lane == 0) {
        unsigned long long* ct = reinterpret_cast<unsigned long long*>(st.counters + h * 8 + 3);
        if (a) atomicAdd(ct + 0, (unsigned long long)a);
        if (bq) atomicAdd(ct + 1, (unsigned long long)bq);
        if (c) atomicAdd(ct + 2, (unsigned long long)c);
      }
    }
    vbytes = warp_sum_ll(vbytes);
    if (lane == 0)
      atomicAdd(reinterpret_cast<unsigned long long*>(st.unit_bytes + (size_t)u * 4 + 1), (unsigned long long)vbytes);
    __syncwarp();
  }
  if (lane == 0) {
    __threadfence();
    const unsigned done = atomicAdd(st.work + 3, 1u);
    if (done == gridDim.x * 4 - 1) {
      st.work[2] = 0;
      st.work[3] = 0;
      __threadfence();
    }
  }
}

// o = o_est + sum over the unit's pages of o_partial, fixed order (deterministic).
__global__ void __launch_bounds__(128) combine_kernel(akv_store_t s, akv_cfg_t cfg, akv_step_t st) {
  const int h = blockIdx.x;
  const int u = h / cfg.group;
  const int n = s.lengths[u];
  const int npg = (n + P - 1) / P;
  const float* part = st.o_partial + (size_t)h * s.max_pages * D + threadIdx.x;
  float acc = st.o_est[(size_t)h * D + threadIdx.x];
  int pg = 0;
  for (; pg + 4 <= npg; pg += 4) {
    const float a = part[(pg + 0) * D], b = part[(pg + 1) * D], c = part[(pg + 2) * D], d = part[(pg + 3) * D];
    acc += ((a + b) + (c + d));
  }
  for (; pg < npg; ++pg) acc += part[pg * D];
  st.o[(size_t)h * D + threadIdx.x] = acc;
}

template <typename K>
static int resident_blocks_pv(K kernel, size_t smem) {
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, 128, smem);
  return std::max(1, sms * std::max(per, 1));
}

template <int G, bool TRUNC, bool EXPORT>
static void launch_pv_t(const akv_store_t& s, const akv_cfg_t& cfg, const akv_step_t& st, int max_len,
                        cudaStream_t stream) {
  const size_t smem = 4 * sizeof(PvWarp<G>);
  static int resident = 0;
  if (!resident) {
    cudaFuncSetAttribute(pv_kernel<G, TRUNC, EXPORT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    resident = resident_blocks_pv(pv_kernel<G, TRUNC, EXPORT>, smem);
  }
  const int cap = s.max_pages * P;
  const int npg = (max_len + P - 1) / P;
  const long long items = (long long)s.n_units * npg;
  const int grid = (int)std::min<long long>(resident, (items + 3) / 4);
  pv_kernel<G, TRUNC, EXPORT><<<std::max(grid, 1), 128, smem, stream>>>(s, cfg, st, cap, npg);
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
  combine_kernel<<<s.n_units * cfg.group, D, 0, stream>>>(s, cfg, st);
}

}  // namespace akv
