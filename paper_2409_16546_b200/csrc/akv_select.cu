// softmax + estimate_output (D3) +
// rule2_targets for every (unit, q-head): one CTA each.
//
//  1. combine the per-32-token-chunk (max, sum exp) of the QK kernel -> M, L;
//  2. p_t = exp(s_t - M) * (1/L) (written to probs); tokens with
//     p_t >= pmax * 2^-m are compacted into a shared candidate list
//     (warp-aggregated atomics); with 256-thread CTAs (contexts <= 8k) the
//     per-token fetch-plan bound of step 6 is computed here as well;
//  3. |C| <= k_sel: the selection is C.  Otherwise the k_sel largest by
//     (p desc, t asc): an exact 4-pass radix select on the fp32 bit patterns
//     of the candidates (p >= 0, so bit order = value order), ties at the
//     k-th value resolved by ascending t;
//  4. the selection is sorted by t; o_est = sum_{t in sel} p_t * V[t] at T16
//     (warps split the rows, fixed-order reduction);
//  5. target_r = floor(log2|o_est_r|) - 10 (0 -> unknown) plus the minimum
//     known target and an any-unknown flag for the PV superset rule (H6);
//  6. the PV fetch plan: per-row need-mid / need-low bitmaps.
// CTA size: 256 threads up to 8k tokens, 512 above (launch_select).
#include "akv_common.cuh"

namespace akv {

constexpr int SW = 8;      // warps that run the digit scan and the o_est gather (fixed: results independent of ST)
constexpr int CAND = 2048; // shared candidate capacity (overflow -> global fallback scan)

template <int ST>
struct SelSmem {
  unsigned hist[256];
  int cand_t[CAND];
  float cand_p[CAND];
  int sel[AKV_MAX_KSEL];
  int sel_sorted[AKV_MAX_KSEL];
  float part[SW][D];
  float M, L;
  int ncand, nsel, need_eq, neq;
  unsigned vstar;
  unsigned wsum[SW];
  int wfirst[SW];
  int sel_page[AKV_MAX_KSEL];
  int tmin[4], tunk[4];
  // ST = 256 (max_len <= 8192): the per-token fetch-plan bound of step 6, computed in
  // step 2 next to p (no reload of p / RowMax), and the selection bitmap
  int16_t xs[ST == 256 ? 8192 : 1];
  uint32_t selw[ST == 256 ? 8192 / 32 : 1];
};

// xs sentinels: p = 0 (never fetched unless the row strategy has unknown targets),
// row strategy with RowMax = 0 (T8)
constexpr int16_t XS_P0 = -32768, XS_RM0 = -32767;

__device__ __forceinline__ uint32_t v_word_exact(const uint8_t* vp, int tt, int r) {
  const uint32_t head = vp[tt * D + r];
  const int byte = tt * (D / 2) + (r >> 3) * 4 + (r & 3);
  const uint32_t mb = vp[MID + byte], lb = vp[LOW + byte];
  const bool first = (r & 7) < 4;
  const uint32_t mid = first ? (mb >> 4) : (mb & 0xF);
  const uint32_t low = first ? (lb & 0xF) : (lb >> 4);
  return (head << 8) | (mid << 4) | low;
}

template <int ST>
__global__ void __launch_bounds__(ST, ST == 256 ? 4 : 2) select_kernel(akv_store_t s, akv_cfg_t cfg, akv_step_t st,
                                                                    int cap) {
  pdl_trigger();
  pdl_wait();
  const int h = blockIdx.x;
  const int G = cfg.group;
  const int u = h / G;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = s.lengths[u];
  const int nch = (n + 31) / 32;  // 32-token chunks with (max, sum exp) from the QK kernel
  __shared__ SelSmem<ST> sm;

  // the first batch of scores is loaded before the statistics are known (overlaps step 1)
  constexpr int BT = 8;
  const float* sc = st.scores + (size_t)h * cap;
  constexpr bool FASTNEED = ST == 256;
  const uint16_t* rmu = s.rowmax + (size_t)u * s.max_pages * P;
  float sv0[BT];
  uint32_t rm0[BT];
#pragma unroll
  for (int b = 0; b < BT; ++b) {
    const int t = b * ST + tid;
    sv0[b] = t < n ? sc[t] : 0.f;
    rm0[b] = FASTNEED && t < n ? (uint32_t)rmu[t] : 0u;
  }

  // 1. global softmax statistics (fixed assignment + butterfly: deterministic); the
  //    chunk pairs are read once (up to 8 per lane) and reused for the second pass
  if (warp == 0) {
    const float2* ps = reinterpret_cast<const float2*>(st.page_stats) + (size_t)h * s.max_pages * (P / 32);
    constexpr int CR = 8;
    float2 cv[CR];
#pragma unroll
    for (int r = 0; r < CR; ++r) cv[r] = lane + 32 * r < nch ? ps[lane + 32 * r] : make_float2(-INFINITY, 0.f);
    float m = -INFINITY;
#pragma unroll
    for (int r = 0; r < CR; ++r) m = fmaxf(m, cv[r].x);
    for (int i = lane + 32 * CR; i < nch; i += 32) m = fmaxf(m, ps[i].x);
    m = warp_max(m);
    float l = 0.f;
#pragma unroll
    for (int r = 0; r < CR; ++r)
      if (lane + 32 * r < nch) l += cv[r].y * expf(cv[r].x - m);
    for (int i = lane + 32 * CR; i < nch; i += 32) {
      const float2 v = ps[i];
      l += v.y * expf(v.x - m);
    }
    l = warp_sum(l);
    if (lane == 0) {
      sm.M = m;
      sm.L = l;
      sm.ncand = 0;
      sm.nsel = 0;
      sm.neq = 0;
    }
  }
  __syncthreads();
  const float M = sm.M, L = sm.L;
  const float invL = 1.0f / L;
  const float pmax = invL;  // = expf(0) / L, the argmax token's p
  const float thr = ldexpf(pmax, -cfg.m);
  const bool est = cfg.force_tier == 0 && cfg.trunc_bits == 0 && cfg.k_sel > 0;  // k_sel = 0: softmax only
  const int k_sel = max(min(cfg.k_sel, AKV_MAX_KSEL), 1);
  float* pr = st.probs + (size_t)h * cap;
  uint32_t* bits = st.sel_bits + (size_t)h * (cap >> 5);

  // 2. probabilities, bitmap reset, candidate compaction: batches of BT tokens per thread,
  //    the next batch's scores (and RowMax words) loaded before the current one is used.
  //    p = exp(s - M) * (1/L): one rounding more than a division (~1 ulp, far inside the
  //    2^-18 knife-edge margin of D11) and no division slow path.
  for (int w = tid; w < (n + 31) / 32; w += ST) {
    bits[w] = 0u;
    if (FASTNEED) sm.selw[w] = 0u;
  }
  const float* scb = sc + tid;
  const uint16_t* rmb = rmu + tid;
  float* prb = pr + tid;
  for (int t0 = 0; t0 < n; t0 += ST * BT) {
    float sv[BT];
    uint32_t rmv[BT];
#pragma unroll
    for (int b = 0; b < BT; ++b) {
      sv[b] = sv0[b];
      rmv[b] = rm0[b];
    }
    const int t1 = t0 + ST * BT;
    if (t1 < n) {
      if (t1 + ST * BT <= n) {
#pragma unroll
        for (int b = 0; b < BT; ++b) {
          sv0[b] = scb[t1 + b * ST];
          rm0[b] = FASTNEED ? (uint32_t)rmb[t1 + b * ST] : 0u;
        }
      } else {
#pragma unroll
        for (int b = 0; b < BT; ++b) {
          const bool in = t1 + b * ST + tid < n;
          sv0[b] = in ? scb[t1 + b * ST] : 0.f;
          rm0[b] = FASTNEED && in ? (uint32_t)rmb[t1 + b * ST] : 0u;
        }
      }
    }
#pragma unroll
    for (int b = 0; b < BT; ++b) {
      const int t = t0 + b * ST + tid;
      const bool in = t < n;
      const float p = expf(sv[b] - M) * invL;
      const bool cand = in && est && p >= thr;
      if (in) {
        prb[t0 + b * ST] = p;
        if (FASTNEED) {
          const uint32_t rm = rmv[b];
          int x;
          if (p == 0.f) x = XS_P0;
          else if (cfg.strategy == 1) x = rm == 0 ? XS_RM0 : floor_log2f(p) + magexp16(rm) + cfg.margin_bits;
          else x = floor_log2f(p) + max(bexp16(rm), 1) - 15 + cfg.margin_bits;
          sm.xs[t] = (int16_t)x;
        }
      }
      const unsigned bb = __ballot_sync(0xFFFFFFFFu, cand);
      if (bb) {
        int base = 0;
        if (lane == 0) base = atomicAdd(&sm.ncand, __popc(bb));
        base = __shfl_sync(0xFFFFFFFFu, base, 0);
        const int slot = base + __popc(bb & ((1u << lane) - 1u));
        if (cand && slot < CAND) {
          sm.cand_t[slot] = t;
          sm.cand_p[slot] = p;
        }
      }
    }
  }
  if (tid < 256) sm.hist[tid] = 0;
  __syncthreads();
  const int ncand = sm.ncand;

  if (est) {
    if (ncand <= k_sel) {
      // 3a. every candidate is selected
      for (int i = tid; i < ncand; i += ST) sm.sel[i] = sm.cand_t[i];
      if (tid == 0) sm.nsel = ncand;
    } else {
      // 3b. radix select of the k_sel-th largest key among the candidates
      const bool shared_list = ncand <= CAND;
      unsigned prefix = 0, mask = 0;
      int k = k_sel;
      for (int shift = 24; shift >= 0; shift -= 8) {
        if (shared_list) {
          for (int i = tid; i < ncand; i += ST) {
            const unsigned key = __float_as_uint(sm.cand_p[i]);
            if ((key & mask) == prefix) atomicAdd(&sm.hist[(key >> shift) & 0xFF], 1u);
          }
        } else {
          for (int t = tid; t < n; t += ST) {
            const float p = pr[t];
            const unsigned key = __float_as_uint(p);
            if (p >= thr && (key & mask) == prefix) atomicAdd(&sm.hist[(key >> shift) & 0xFF], 1u);
          }
        }
        __syncthreads();
        {
          // digit of the k-th largest key: scan the histogram from the top bin down
          // (threads 0..255: thread t owns bin 255 - t; block-wide scan by warp shuffles)
          const bool scan = tid < 256;
          const unsigned hv = scan ? sm.hist[255 - tid] : 0u;
          unsigned incl = hv;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += y;
          }
          if (scan && lane == 31) sm.wsum[warp] = incl;
          __syncthreads();
          unsigned before = 0;
          if (scan)
            for (int w = 0; w < warp; ++w) before += sm.wsum[w];
          incl += before;
          const bool hit = scan && ((int)incl >= k || tid == 255);
          const unsigned hb = __ballot_sync(0xFFFFFFFFu, hit);
          if (scan && lane == 0) sm.wfirst[warp] = hb ? warp * 32 + __ffs(hb) - 1 : 0x7FFFFFFF;
          __syncthreads();
          int first = 0x7FFFFFFF;
#pragma unroll
          for (int w = 0; w < SW; ++w) first = min(first, sm.wfirst[w]);
          if (tid == first) {
            sm.need_eq = k - (int)(incl - hv);
            sm.vstar = prefix | ((unsigned)(255 - tid) << shift);
          }
        }
        __syncthreads();
        k = sm.need_eq;
        prefix = sm.vstar;
        mask |= 0xFFu << shift;
        if (tid < 256) sm.hist[tid] = 0;
        __syncthreads();
      }
      const unsigned vstar = sm.vstar;
      const int need_eq = sm.need_eq;
      // keys > v* are all selected (fewer than k_sel); keys == v*: the need_eq smallest t
      auto visit = [&](int t, float p) {
        const unsigned key = __float_as_uint(p);
        if (key > vstar) {
          const int slot = atomicAdd(&sm.nsel, 1);
          sm.sel[slot] = t;
        } else if (key == vstar) {
          const int slot = atomicAdd(&sm.neq, 1);
          if (slot < CAND) sm.cand_t[slot] = t;  // reuse the candidate buffer (already consumed)
        }
      };
      __syncthreads();
      if (shared_list) {
        // copy out first (visit overwrites cand_t)
        int my_t[CAND / ST];
        float my_p[CAND / ST];
        int cnt = 0;
        for (int i = tid; i < ncand; i += ST, ++cnt) {
          my_t[cnt] = sm.cand_t[i];
          my_p[cnt] = sm.cand_p[i];
        }
        __syncthreads();
        for (int i = 0; i < cnt; ++i) visit(my_t[i], my_p[i]);
      } else {
        for (int t = tid; t < n; t += ST) {
          const float p = pr[t];
          if (p >= thr) visit(t, p);
        }
      }
      __syncthreads();
      // the need_eq smallest t among the ties (rank by counting; ties are rare)
      const int neq = min(sm.neq, CAND);
      const int base = sm.nsel;
      for (int i = tid; i < neq; i += ST) {
        const int t = sm.cand_t[i];
        int rank = 0;
        for (int j = 0; j < neq; ++j) rank += sm.cand_t[j] < t;
        if (rank < need_eq) sm.sel[base + rank] = t;
      }
      __syncthreads();
      if (tid == 0) sm.nsel = base + min(need_eq, neq);
    }
  }
  __syncthreads();
  const int cnt = est ? min(sm.nsel, AKV_MAX_KSEL) : 0;

  // 4. sort the selection by t (rank by counting, <= 64 entries), bitmap, o_est
  if (tid < cnt) {
    const int t = sm.sel[tid];
    int rank = 0;
    for (int j = 0; j < cnt; ++j) rank += sm.sel[j] < t;
    sm.sel_sorted[rank] = t;
    sm.sel_page[rank] = s.page_table[(size_t)u * s.max_pages + t / P];
    atomicOr(bits + (t >> 5), 1u << (t & 31));
    if (FASTNEED) atomicOr(&sm.selw[t >> 5], 1u << (t & 31));
  }
  __syncthreads();
  // rows split over warps (warp w: rows w, w+8, ...), lane = 4 channels; fixed-order reduction.
  // Every row's words and p are loaded before the (in-order) accumulation.
  {
    constexpr int RW = 4;  // rows loaded together (per warp: rows warp + 8r)
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int r0 = 0; warp < SW && warp + r0 * SW < cnt; r0 += RW) {
      float pv[RW];
      uint32_t wv[RW][4];
#pragma unroll
      for (int r = 0; r < RW; ++r) {
        const int i = warp + (r0 + r) * SW;
        pv[r] = 0.f;
        wv[r][0] = wv[r][1] = wv[r][2] = wv[r][3] = 0u;
        if (i < cnt) {
          const int t = sm.sel_sorted[i];
          const uint8_t* vp = s.v_pool + (size_t)sm.sel_page[i] * PAGE;
          pv[r] = pr[t];
#pragma unroll
          for (int e = 0; e < 4; ++e) wv[r][e] = v_word_exact(vp, t % P, lane * 4 + e);
        }
      }
#pragma unroll
      for (int r = 0; r < RW; ++r) {
        if (warp + (r0 + r) * SW < cnt) {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            acc[e] = fmaf(pv[r], __half2float(__ushort_as_half((unsigned short)wv[r][e])), acc[e]);
        }
      }
    }
    if (warp < SW) {
#pragma unroll
      for (int e = 0; e < 4; ++e) sm.part[warp][lane * 4 + e] = acc[e];
    }
  }
  __syncthreads();
  if (tid < D) {
    const int r = tid;
    float o = 0.f;
#pragma unroll
    for (int w = 0; w < SW; ++w) o += sm.part[w][r];
    st.o_est[(size_t)h * D + r] = o;
    const bool known = o != 0.f;
    const int tg = known ? floor_log2f(o) - 10 : AKV_TARGET_UNKNOWN;
    st.targets[(size_t)h * D + r] = tg;
    const int wmin = warp_min_i(known ? tg : INT_MAX);
    const int wunk = warp_sum_i(known ? 0 : 1);
    if (lane == 0) {
      sm.tmin[warp] = wmin;
      sm.tunk[warp] = wunk;
    }
    if (r < cnt) st.sel_idx[(size_t)h * AKV_MAX_KSEL + r] = sm.sel_sorted[r];
  }
  __syncthreads();
  const int tmin_all = min(min(sm.tmin[0], sm.tmin[1]), min(sm.tmin[2], sm.tmin[3]));
  const int unk_all = sm.tunk[0] + sm.tunk[1] + sm.tunk[2] + sm.tunk[3];
  // 6. V rows needing the mid / low nibble row for this head (PV fetch plan):
  //    element strategy: RowMax superset bound (H6); row strategy: the row tier (D7)
  if (FASTNEED) {
    // from the bounds of step 2: bound - tmin > 2 (mid) / > 6 (low), i.e. the row tier >= 12 / 16
    uint32_t* nb = st.need_bits + (size_t)h * 2 * (cap >> 5);
    for (int w = warp; w < (n + 31) / 32; w += ST / 32) {
      const int t = 32 * w + lane;
      bool nm = false, nlw = false;
      if (t < n && est) {
        const int x = sm.xs[t];
        if (cfg.strategy == 1) {
          if (unk_all) nm = nlw = true;
          else if (x != XS_P0 && x != XS_RM0) {
            nm = x - tmin_all > 2;
            nlw = x - tmin_all > 6;
          }
        } else {
          // an unknown target (o_est_r == 0) forces T16 on every read contributing to that
          // dim, p_t == 0 included (Appendix A D5 as amended in DESIGN §4)
          nm = unk_all || (x != XS_P0 && x - tmin_all > 2);
          nlw = unk_all || (x != XS_P0 && x - tmin_all > 6);
        }
      }
      const uint32_t sw = sm.selw[w];
      const unsigned bm = __ballot_sync(0xFFFFFFFFu, nm) & ~sw, bl = __ballot_sync(0xFFFFFFFFu, nlw) & ~sw;
      if (lane == 0) {
        nb[w] = bm;
        nb[(cap >> 5) + w] = bl;
      }
    }
  } else {
    uint32_t* nb = st.need_bits + (size_t)h * 2 * (cap >> 5);
    for (int t0 = 0; t0 < n; t0 += ST * BT) {
      float pv[BT];
      uint32_t rmv[BT], selw[BT];
#pragma unroll
      for (int b = 0; b < BT; ++b) {
        const int t = t0 + b * ST + tid;
        const bool in = t < n && est;
        pv[b] = in ? pr[t] : 0.f;
        rmv[b] = in ? (uint32_t)s.rowmax[(size_t)u * s.max_pages * P + t] : 0u;
        selw[b] = in ? bits[t >> 5] : 0u;
      }
#pragma unroll
      for (int b = 0; b < BT; ++b) {
        const int t = t0 + b * ST + tid;
        bool nm = false, nlw = false;
        if (t < n && est) {
          const bool sel = (selw[b] >> (t & 31)) & 1u;
          const float p = pv[b];
          const uint32_t rm = rmv[b];
          if (!sel && cfg.strategy == 1) {
            int tier = 16;
            if (!unk_all) {
              if (p == 0.f || rm == 0) tier = 8;
              else {
                const int tr = min(max(floor_log2f(p) + magexp16(rm) + 1 - tmin_all - 1 + cfg.margin_bits, 0), 10);
                tier = tr <= 2 ? 8 : (tr <= 6 ? 12 : 16);
              }
            }
            nm = tier >= 12;
            nlw = tier == 16;
          } else if (!sel) {
            if (unk_all) {
              nm = nlw = true;  // SPEC.md:169, p_t == 0 included
            } else if (p > 0.f) {
              const int bound = floor_log2f(p) + (max(bexp16(rm), 1) - 15) + 1 - tmin_all - 1 + cfg.margin_bits;
              nm = bound > 2;
              nlw = bound > 6;
            }
          }
        }
        const unsigned bm = __ballot_sync(0xFFFFFFFFu, nm), bl = __ballot_sync(0xFFFFFFFFu, nlw);
        if (lane == 0 && t < n) {
          nb[t >> 5] = bm;
          nb[(cap >> 5) + (t >> 5)] = bl;
        }
      }
    }
  }
  if (tid == 0) {
    const int tmin = tmin_all;
    const int unk = unk_all;
    int32_t* hm = st.head_meta + (size_t)h * 4;
    hm[0] = cnt;
    hm[1] = tmin;
    hm[2] = est ? (unk > 0) : 0;
    hm[3] = n;
    float* hf = st.head_metaf + (size_t)h * 4;
    hf[0] = M;
    hf[1] = L;
    hf[2] = pmax;
    hf[3] = thr;
    int64_t* ct = st.counters + (size_t)h * 8;
    ct[3] = 0;
    ct[4] = 0;
    ct[5] = (int64_t)cnt * D;  // estimation reads at T16, counted once (D6)
    if (cnt) atomicAdd(reinterpret_cast<unsigned long long*>(st.unit_bytes + (size_t)u * 4 + 1),
                       (unsigned long long)cnt * 2 * D);
  }
}

void launch_select(const akv_store_t& s, const akv_cfg_t& cfg, const akv_step_t& st, int max_len, cudaStream_t stream) {
  const int cap = s.max_pages * P;
  // long contexts: more threads per head (the per-head chain is the latency); 512 threads
  // keep 2 CTAs per SM, so up to 296 heads run in one wave (c4: 1024 threads 47 us, 512: 43 us)
  // a grid of more than one wave is launched without PDL: early-launched CTAs of the first wave
  // squat on SMs through the previous kernel's tail and the second wave starts late (c3, 1024
  // heads over 592 slots: 256.5 -> 239.5 us per step; one-wave grids keep PDL: c2 144.1 vs 145.7)
  const int heads = s.n_units * cfg.group;
  if (max_len > 8192) {
    const int res = resident_ctas<select_kernel<512>>(512, 0);
    launch_pdl(heads > res ? PDL_OFF : PDL_SELECT, select_kernel<512>, dim3(heads), dim3(512), 0, stream, s, cfg, st, cap);
  } else {
    const int res = resident_ctas<select_kernel<256>>(256, 0);
    launch_pdl(heads > res ? PDL_OFF : PDL_SELECT, select_kernel<256>, dim3(heads), dim3(256), 0, stream, s, cfg, st, cap);
  }
}

}  // namespace akv
