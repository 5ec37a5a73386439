// output_aligned for every (unit, q-head).
//
// Warp-specialised persistent kernel, one CTA per SM, 6-stage shared ring of
// half pages (128 V rows: 16 KB head rows + up to 8 KB mid + 8 KB low rows +
// the rows' metadata), two half-page stages per page:
//
//  producer warp   walks a contiguous range of (unit, page) items, reads the
//                  page's per-head "need mid / need low" row bitmaps written by
//                  akv_softmax_select (RowMax superset rule; row
//                  tiers for the row strategy, D7) one page ahead, and fills
//                  each stage: the head rows by one TMA bulk copy; only the
//                  64 B mid / low rows some q-head of the kv-head needs, and
//                  the per-row metadata (p_t, selection bits, need bits,
//                  rule-2 targets), by cp.async from all 32 lanes;
//  8 consumer      warps: 16 lanes per row x 8 channels per lane, two rows per
//                  warp instruction, 16 rows per warp per half page.  A per-half
//                  pre-pass folds the selection (D6: selected rows' T16
//                  contribution is already in o_est) and the page end into p.
//                  A 16-row block that no q-head needs beyond T8 takes a
//                  branch-free unrolled path (4 PRMT per 8 elements); other
//                  rows apply each head's rule: p_t = 0 -> T8 (D5); ELEMENT:
//                  keep mid iff max(bexp,1) + e(p_t) > 17 + target_r - margin,
//                  low iff > that + 4 (D4); row strategy: the row tier (D7);
//                  forced / baseline tiers.  Truncation is applied after the
//                  fetch, so the masks equal the oracle's bit for bit.  fp16 ->
//                  fp32 by HADD2.F32 and p_t * V~ by the packed FFMA2 into fp32
//                  (SPEC.md:379).
// The page's partial output goes to o_partial[h][page]; akv_combine adds o_est
// and the partials in a fixed order (deterministic).
#include <algorithm>

#include "akv_common.cuh"

namespace akv {

constexpr int HR = P / 2;                // rows per half page
constexpr int VS = HR * D * 2;           // 32 KB: head [128][128] | mid [128][64] | low [128][64]
constexpr int VS_MID = HR * D, VS_LOW = HR * D + HR * (D / 2);

template <int G>
struct PvShape {
  static constexpr int NS = G >= 4 ? 4 : 6;  // ring stages (half pages; shared memory bound for G >= 4)
  static constexpr int PRODUCERS = 2;          // producer warp h fills the half-page stages of half h
  static constexpr int THREADS = 32 * (PRODUCERS + 8);
};

template <int G>
struct alignas(16) PvAux {  // per-row / per-head metadata of one half page (cp.async)
  float probs[G][HR];
  int32_t targets[G][D];
  uint32_t sel[G][4];
  uint32_t need[G][2][4];
};

struct alignas(16) PvMeta {
  int item, u, pg, n;
  int half, rows, pad0, pad1;     // rows valid in this half
  uint32_t un_mid[4], un_low[4];  // union over q-heads of the need bitmaps of this half
};

template <int G>
struct alignas(128) PvSmem {
  uint8_t data[PvShape<G>::NS][VS];
  PvAux<G> aux[PvShape<G>::NS];
  PvMeta meta[PvShape<G>::NS];
  float red[2][8][G][D];  // per-warp partial outputs, double-buffered (one barrier per page)
  uint64_t full[PvShape<G>::NS], empty[PvShape<G>::NS];
};

__device__ __forceinline__ bool bitw(const uint32_t* w, int r) { return (w[r >> 5] >> (r & 31)) & 1u; }

__device__ __forceinline__ void t8_words(uint2 h, uint32_t w[4]) {
  const uint32_t c80 = 0x80808080u;
  w[0] = prmt(h.x, c80, 0x1404);
  w[1] = prmt(h.x, c80, 0x3424);
  w[2] = prmt(h.y, c80, 0x1404);
  w[3] = prmt(h.y, c80, 0x3424);
}

// ----------------------------------------------------------------------------
// producer
// ----------------------------------------------------------------------------
struct PvPage {
  int u, n;
  size_t pid;       // pool page id
  uint32_t um, ul;  // lane w < 8: union need words w of the page
};

template <int G>
__device__ __forceinline__ void pv_fetch(PvPage& f, const akv_cfg_t& cfg, const akv_step_t& st, int u, int pg,
                                         int n, int cap, bool uniform) {
  const int lane = threadIdx.x & 31;
  f.u = u;
  f.n = n;
  f.um = f.ul = 0u;
  if (lane < 8) {
    if (uniform) {
      f.um = cfg.force_tier >= 12 || cfg.trunc_bits ? 0xFFFFFFFFu : 0u;
      f.ul = cfg.force_tier >= 16 || cfg.trunc_bits ? 0xFFFFFFFFu : 0u;
    } else {
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const uint32_t* nb = st.need_bits + ((size_t)u * G + j) * 2 * (cap >> 5) + pg * 8 + lane;
        f.um |= nb[0];
        f.ul |= nb[cap >> 5];
      }
    }
  }
}

template <int G>
__device__ void pv_stage(PvSmem<G>& sm, int stage, int hf, int item, int pg, const PvPage& f, const akv_store_t& s,
                         const akv_step_t& st, int cap) {
  const int lane = threadIdx.x & 31;
  PvMeta& mt = sm.meta[stage];
  const int rows = min(max(f.n - pg * P - hf * HR, 0), HR);
  // this half's need words (rows beyond n hold stale bits)
  uint32_t um[4], ul[4];
  {
    const int lo = (lane & 7) * 32, valid = min(max(f.n - pg * P - lo, 0), 32);
    const uint32_t vm = valid >= 32 ? 0xFFFFFFFFu : ((1u << valid) - 1u);
    const uint32_t m0 = f.um & vm, l0 = f.ul & vm;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      um[w] = __shfl_sync(0xFFFFFFFFu, m0, 4 * hf + w);
      ul[w] = __shfl_sync(0xFFFFFFFFu, l0, 4 * hf + w);
    }
  }
  int nm = 0, nl = 0;
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    nm += __popc(um[w]);
    nl += __popc(ul[w]);
  }
  if (lane == 0) {
    mt.item = item;
    mt.u = f.u;
    mt.pg = pg;
    mt.n = f.n;
    mt.half = hf;
    mt.rows = rows;
  }
  if (lane < 4) {
    uint32_t a = um[0], b = ul[0];
#pragma unroll
    for (int w = 1; w < 4; ++w)
      if (lane == w) {
        a = um[w];
        b = ul[w];
      }
    mt.un_mid[lane] = a;
    mt.un_low[lane] = b;
  }
  const uint8_t* src = s.v_pool + f.pid * PAGE;
  uint8_t* dst = sm.data[stage];
  PvAux<G>& ax = sm.aux[stage];
  __syncwarp();
#if AKV_PROBE == 2  // measurement aid: no plane loads (consumer-bound time)
  if (lane == 0) {
    mbar_arrive(&sm.full[stage]);
#else
  if (lane == 0) {
    // head rows of this half: one TMA bulk copy
    mbar_arrive_expect_tx(&sm.full[stage], (uint32_t)rows * D);
    if (rows) bulk_g2s(dst, src + hf * HR * D, (uint32_t)rows * D, &sm.full[stage]);
#endif
    const uint32_t vbytes = (uint32_t)rows * D + (uint32_t)(nm + nl) * (D / 2);
    atomicAdd(reinterpret_cast<unsigned long long*>(st.unit_bytes + (size_t)f.u * 4 + 1), (unsigned long long)vbytes);
  }
  // nibble rows (64 B) and per-row metadata: cp.async from all lanes
#if AKV_PROBE != 2
  cp_rows<4, D / 2>(um, dst + VS_MID, src + MID + hf * HR * (D / 2));
  cp_rows<4, D / 2>(ul, dst + VS_LOW, src + LOW + hf * HR * (D / 2));
#endif
#pragma unroll
  for (int j = 0; j < G; ++j) {
    const size_t h = (size_t)f.u * G + j;
    const uint8_t* pr = reinterpret_cast<const uint8_t*>(st.probs + h * cap + (size_t)pg * P + hf * HR);
    cp_async16(reinterpret_cast<uint8_t*>(ax.probs[j]) + lane * 16, pr + lane * 16);
    cp_async16(reinterpret_cast<uint8_t*>(ax.targets[j]) + lane * 16,
               reinterpret_cast<const uint8_t*>(st.targets + h * D) + lane * 16);
    const uint32_t* selp = st.sel_bits + h * (cap >> 5) + pg * 8 + hf * 4;
    const uint32_t* nbp = st.need_bits + h * 2 * (cap >> 5) + pg * 8 + hf * 4;
    if (lane == 0) cp_async16(ax.sel[j], selp);
    else if (lane == 1) cp_async16(ax.need[j][0], nbp);
    else if (lane == 2) cp_async16(ax.need[j][1], nbp + (cap >> 5));
  }
  cp_async_arrive_noinc(&sm.full[stage]);
}

// ----------------------------------------------------------------------------
// consumer
// ----------------------------------------------------------------------------
template <int G, bool TRUNC, bool EXPORT>
__device__ __forceinline__ void pv_consume_half(PvSmem<G>& sm, int stage, int w8, const akv_cfg_t& cfg,
                                                const akv_step_t& st, int cap, float2 (&acc)[G][4],
                                                int (&adj)[G][3]) {
  const int lane = threadIdx.x & 31;
  const int half = lane >> 4, cl = lane & 15;
  const PvMeta& mt = sm.meta[stage];
  PvAux<G>& ax = sm.aux[stage];
  const uint8_t* pgd = sm.data[stage];
  const int u = mt.u, pg = mt.pg, hf = mt.half, rows = mt.rows;
  const bool aligned = cfg.force_tier == 0 && !TRUNC;
  const int uni = TRUNC ? 16 : cfg.force_tier;
  uint32_t tkm = 0xFFFFFFFFu, tf = 0u;
  if (TRUNC) {
    const int kb = cfg.trunc_bits - 6;
    const uint32_t km = (0xFFFFu << (10 - kb)) & 0xFFFFu;
    const uint32_t fill = kb < 10 ? (1u << (9 - kb)) : 0u;
    tkm = km | (km << 16);
    tf = fill | (fill << 16);
  }
  uint8_t* vt = (EXPORT && st.v_tiers)
                    ? st.v_tiers + ((size_t)u * G * cap + (size_t)pg * P + (size_t)hf * HR) * D + cl * 8
                    : nullptr;
  const int r0 = w8 * 16;  // this warp's 16 rows inside the half

  // base counts: every valid unselected row at T8 (aligned) or at the uniform tier
  if (w8 == 0 && lane < G) {
#pragma unroll
    for (int j = 0; j < G; ++j) {
      if (j != lane) continue;
      int nsel = 0;
      if (aligned) {
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const int valid = min(max(rows - w * 32, 0), 32);
          const uint32_t vm = valid >= 32 ? 0xFFFFFFFFu : ((1u << valid) - 1u);
          nsel += __popc(ax.sel[j][w] & vm);
        }
      }
      const int base = (rows - nsel) * D;
      if (aligned || uni == 8) adj[j][0] += base;
      else if (uni == 12) adj[j][1] += base;
      else adj[j][2] += base;
    }
  }
  if (r0 >= rows) return;
  // pre-pass: fold the selection (D6) and the page end into p (0 -> no contribution)
  if (lane < 16) {
    const int r = r0 + lane;
#pragma unroll
    for (int j = 0; j < G; ++j)
      if (r >= rows || (aligned && bitw(ax.sel[j], r))) ax.probs[j][r] = 0.f;
  }
  __syncwarp();
  const bool full_blk = r0 + 16 <= rows;
  if (aligned && full_blk && ((mt.un_mid[r0 >> 5] >> (r0 & 31)) & 0xFFFFu) == 0) {
    // fast block: every row is T8 (or p = 0) for every q-head
    const uint8_t* hp = pgd + (r0 + half) * D + cl * 8;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint2 h = *reinterpret_cast<const uint2*>(hp + i * 2 * D);
      uint32_t w[4];
      t8_words(h, w);
      float2 f[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) f[k] = half2_bits_to_float2(w[k]);
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const float p = ax.probs[j][r0 + 2 * i + half];
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[j][k] = ffma2_scalar(f[k], p, acc[j][k]);
        if (EXPORT && vt) {
          const int r = r0 + 2 * i + half;
          const uint32_t c = bitw(ax.sel[j], r) ? 0x10101010u : 0x08080808u;
          *reinterpret_cast<uint2*>(vt + j * (size_t)cap * D + (size_t)r * D) = make_uint2(c, c);
        }
      }
    }
    return;
  }
  // generic rows
  for (int i = 0; i < 8; ++i) {
    const int r = r0 + 2 * i + half;
    if (r >= rows) continue;
    const uint2 h = *reinterpret_cast<const uint2*>(pgd + r * D + cl * 8);
    const bool nm = bitw(mt.un_mid, r), nl = bitw(mt.un_low, r);
    const uint32_t mv = nm ? *reinterpret_cast<const uint32_t*>(pgd + VS_MID + r * (D / 2) + cl * 4) : 0u;
    const uint32_t lv = nl ? *reinterpret_cast<const uint32_t*>(pgd + VS_LOW + r * (D / 2) + cl * 4) : 0u;
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const float p = ax.probs[j][r];
      int mode;  // 0 skip, 1 element, 8/12/16 uniform tier
      if (!aligned) mode = uni;
      else if (bitw(ax.sel[j], r)) mode = 0;
      else if (!bitw(ax.need[j][0], r)) mode = 8;  // includes p == 0 (D5)
      else if (cfg.strategy == 1) mode = bitw(ax.need[j][1], r) ? 16 : 12;
      else mode = 1;
      uint32_t w[4];
      uint32_t clo = 0, chi = 0;
      if (mode == 0) {
        if (EXPORT && vt)
          *reinterpret_cast<uint2*>(vt + j * (size_t)cap * D + (size_t)r * D) = make_uint2(0x10101010u, 0x10101010u);
        continue;
      } else if (mode != 1) {
        if (mode == 8) {
          t8_words(h, w);
        } else {
          const TierMask tm = tier_mask(mode);
          assemble8(h.x, h.y, bsel(tm.mk, mv, 0x88888888u), bsel(tm.lk, lv, tm.lf), w);
          if (aligned) {
            adj[j][0] -= 8;
            if (mode == 12) adj[j][1] += 8;
            else adj[j][2] += 8;
          }
        }
        if (EXPORT) clo = chi = (uint32_t)mode * 0x01010101u;
      } else {
        assemble8(h.x, h.y, mv, lv, w);
        const int ep = p > 0.f ? floor_log2f(p) : -30000;
        const int4 t0 = *reinterpret_cast<const int4*>(&ax.targets[j][cl * 8]);
        const int4 t1 = *reinterpret_cast<const int4*>(&ax.targets[j][cl * 8 + 4]);
        const int tg[8] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int g = tg[e] == AKV_TARGET_UNKNOWN ? -(1 << 20) : 17 + tg[e] - cfg.margin_bits;
          const uint32_t hbyte = ((e < 4 ? h.x : h.y) >> (8 * (e & 3))) & 0xFFu;
          const int E = max((int)((hbyte >> 2) & 31u), 1) + ep;
          const bool km = E > g, kl = E > g + 4;
          const int sh = 16 * (e & 1);
          uint32_t w16 = (w[e >> 1] >> sh) & 0xFFFFu;
          w16 = kl ? w16 : (km ? ((w16 & 0xFFF0u) | 0x8u) : ((w16 & 0xFF00u) | 0x80u));
          w[e >> 1] = (w[e >> 1] & ~(0xFFFFu << sh)) | (w16 << sh);
          adj[j][0] -= km ? 1 : 0;
          adj[j][1] += (km && !kl) ? 1 : 0;
          adj[j][2] += kl ? 1 : 0;
          if (EXPORT) {
            const uint32_t cd = kl ? 16u : (km ? 12u : 8u);
            if (e < 4) clo |= cd << (8 * e);
            else chi |= cd << (8 * (e - 4));
          }
        }
      }
      if (TRUNC) {
#pragma unroll
        for (int k = 0; k < 4; ++k) w[k] = (w[k] & tkm) | tf;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[j][k] = ffma2_scalar(half2_bits_to_float2(w[k]), p, acc[j][k]);
      if (EXPORT && vt) *reinterpret_cast<uint2*>(vt + j * (size_t)cap * D + (size_t)r * D) = make_uint2(clo, chi);
    }
  }
}

template <int G, bool TRUNC, bool EXPORT>
__global__ void __launch_bounds__(PvShape<G>::THREADS, 1) pv_kernel(akv_store_t s, akv_cfg_t cfg, akv_step_t st,
                                                                    int cap, int npg_max) {
  constexpr int PV_NS = PvShape<G>::NS;
  extern __shared__ __align__(128) uint8_t pv_smem_raw[];
  PvSmem<G>& sm = *reinterpret_cast<PvSmem<G>*>(pv_smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < PV_NS; ++i) {
      mbar_init(&sm.full[i], 33);  // expect_tx arrival + 32 cp.async arrivals
      mbar_init(&sm.empty[i], 8);  // one arrival per consumer warp
    }
    mbar_fence_init();
  }
  __syncthreads();
  const long long total = (long long)s.n_units * npg_max;
  const bool uniform = cfg.force_tier != 0 || TRUNC;

  if (warp < PvShape<G>::PRODUCERS) {
    const int my_hf = warp;  // both producers walk the same pages; producer h stages half h
    // ---------------- producer: contiguous item range, need bits one page ahead ----------------
    const long long per = (total + gridDim.x - 1) / gridDim.x;
    const long long i0 = (long long)blockIdx.x * per, i1 = min(total, i0 + per);
    int k = 0;
    PvPage cur, nxt;
    UnitPages up_cur, up_nxt;  // page-table rows: the current unit and (prefetched) the next
    up_cur.u = -1;
    if (i0 < i1) unit_pages_fetch(up_nxt, s, (int)(i0 / npg_max));
    auto advance = [&](long long from, PvPage& f) -> long long {
      for (long long idx = from; idx < i1; ++idx) {
        const int u = (int)(idx / npg_max), pg = (int)(idx % npg_max);
        if (u != up_cur.u) {
          up_cur = up_nxt;
          if ((long long)(u + 1) * npg_max < i1) unit_pages_fetch(up_nxt, s, u + 1);
        }
        const int n = up_cur.n;
        if (pg * P >= n) continue;
        pv_fetch<G>(f, cfg, st, u, pg, n, cap, uniform);
        f.pid = unit_page(up_cur, s, pg);
        return idx;
      }
      return -1;
    };
    long long nidx = advance(i0, nxt);
    while (nidx >= 0) {
      const long long idx = nidx;
      cur = nxt;
      nidx = advance(idx + 1, nxt);  // prefetch the next page's need bits
      const int pg = (int)(idx % npg_max);
      {
        const int kk = k + my_hf, stage = kk % PV_NS;
        mbar_wait(&sm.empty[stage], ((kk / PV_NS) & 1) ^ 1);
        pv_stage<G>(sm, stage, my_hf, (int)idx, pg, cur, s, st, cap);
        k += 2;
      }
    }
    {
      const int kk = k + my_hf, stage = kk % PV_NS;
      mbar_wait(&sm.empty[stage], ((kk / PV_NS) & 1) ^ 1);
      if (lane == 0) sm.meta[stage].item = -1;
      __syncwarp();
      mbar_arrive(&sm.full[stage]);                 // 32 lane arrivals ...
      if (lane == 0) mbar_arrive(&sm.full[stage]);  // ... + the expect_tx slot
      __syncwarp();
    }
  } else {
    const int w8 = warp - PvShape<G>::PRODUCERS;
    int adj[G][3];  // element-count adjustments relative to "every valid unselected row is T8" (current unit)
    int cur_u = -1;
    auto flush_counts = [&]() {
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const int a = warp_sum_i(adj[j][0]), b = warp_sum_i(adj[j][1]), c = warp_sum_i(adj[j][2]);
        if (lane == 0 && cur_u >= 0) {
          unsigned long long* ct = reinterpret_cast<unsigned long long*>(st.counters + ((size_t)cur_u * G + j) * 8 + 3);
          if (a) atomicAdd(ct + 0, (unsigned long long)(long long)a);
          if (b) atomicAdd(ct + 1, (unsigned long long)(long long)b);
          if (c) atomicAdd(ct + 2, (unsigned long long)(long long)c);
        }
        adj[j][0] = adj[j][1] = adj[j][2] = 0;
      }
    };
#pragma unroll
    for (int j = 0; j < G; ++j) adj[j][0] = adj[j][1] = adj[j][2] = 0;
    for (int kp = 0;; ++kp) {
      float2 acc[G][4];
#pragma unroll
      for (int j = 0; j < G; ++j)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) acc[j][kk] = make_float2(0.f, 0.f);
      int u = 0, pg = 0;
      bool done = false;
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        const int kk = 2 * kp + hf, stage = kk % PV_NS;
        mbar_wait(&sm.full[stage], (kk / PV_NS) & 1);
        if (sm.meta[stage].item < 0) {
          done = true;
          break;
        }
        if (hf == 0) {
          u = sm.meta[stage].u;
          pg = sm.meta[stage].pg;
          if (u != cur_u) {
            flush_counts();
            cur_u = u;
          }
        }
#if AKV_PROBE != 1  // measurement aid: 1 = no consumer compute (load-bound time)
        pv_consume_half<G, TRUNC, EXPORT>(sm, stage, w8, cfg, st, cap, acc, adj);
#endif
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[stage]);  // stage no longer read by this warp
      }
      if (done) break;
      // partial o of the page: half-warps -> warp partial (shared, double-buffered) -> every
      // warp reduces a 16-channel slice over the 8 partials in a fixed order
      const int half = lane >> 4, cl = lane & 15;
      float (*red)[G][D] = sm.red[kp & 1];
#pragma unroll
      for (int j = 0; j < G; ++j) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          acc[j][kk].x += __shfl_xor_sync(0xFFFFFFFFu, acc[j][kk].x, 16);
          acc[j][kk].y += __shfl_xor_sync(0xFFFFFFFFu, acc[j][kk].y, 16);
        }
        if (half == 0) {
          float4* dst = reinterpret_cast<float4*>(&red[w8][j][cl * 8]);
          dst[0] = make_float4(acc[j][0].x, acc[j][0].y, acc[j][1].x, acc[j][1].y);
          dst[1] = make_float4(acc[j][2].x, acc[j][2].y, acc[j][3].x, acc[j][3].y);
        }
      }
      named_bar(1, 256);
      for (int i = lane; i < G * 4; i += 32) {
        const int j = i >> 2, c = w8 * 16 + (i & 3) * 4;
        float4 o = *reinterpret_cast<const float4*>(&red[0][j][c]);
#pragma unroll
        for (int w = 1; w < 8; ++w) {  // fixed order
          const float4 a = *reinterpret_cast<const float4*>(&red[w][j][c]);
          o.x += a.x;
          o.y += a.y;
          o.z += a.z;
          o.w += a.w;
        }
        *reinterpret_cast<float4*>(st.o_partial + (((size_t)u * G + j) * (cap / P) + pg) * D + c) = o;
      }
    }
    flush_counts();
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

template <int G>
constexpr bool pv_smem_fits = sizeof(PvSmem<G>) <= 232448;
static_assert(pv_smem_fits<1> && pv_smem_fits<2> && pv_smem_fits<4> && pv_smem_fits<8>, "PV shared memory > 227 KB");

template <int G, bool TRUNC, bool EXPORT>
static void launch_pv_t(const akv_store_t& s, const akv_cfg_t& cfg, const akv_step_t& st, int max_len,
                        cudaStream_t stream) {
  static int sms = 0;
  const size_t smem = sizeof(PvSmem<G>);
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(pv_kernel<G, TRUNC, EXPORT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  const int cap = s.max_pages * P;
  const int npg = (max_len + P - 1) / P;
  const long long items = (long long)s.n_units * npg;
  const int grid = (int)std::min<long long>(sms, std::max<long long>(items / 2, 1));
  pv_kernel<G, TRUNC, EXPORT><<<grid, PvShape<G>::THREADS, smem, stream>>>(s, cfg, st, cap, npg);
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
