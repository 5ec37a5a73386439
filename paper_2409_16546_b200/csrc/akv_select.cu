// softmax + estimate_output (D3) +
// rule2_targets for every (unit, q-head): one CTA each.
//
//  1. combine the per-page (max, sum exp) of the QK kernel -> M, L;
//  2. p_t = exp(s_t - M) / L  (written to probs, may overwrite scores);
//  3. approximate top-k: C = {t : p_t >= pmax * 2^-m}; if |C| > k_sel keep the
//     k_sel largest by (p desc, t asc) via an exact 4-pass radix select on the
//     fp32 bit patterns (p >= 0, so bit order = value order);
//  4. o_est = sum_{t in sel, ascending t} p_t * V[t] read at T16;
//  5. target_r = floor(log2|o_est_r|) - 10 (0 -> unknown), plus the minimum
//     known target and an any-unknown flag for the PV superset rule (H6).
#include "akv_common.cuh"

namespace akv {

constexpr int ST = 512;  // threads per select CTA

struct SelSmem {
  unsigned hist[256];
  int wcnt[ST / 32][2];
  int sel_idx[AKV_MAX_KSEL];
  float M, L;
  int ncand, sel_count, need_eq;
  unsigned vstar;
  int tmin[4], tunk[4];
};

__device__ __forceinline__ uint32_t v_word_exact(const uint8_t* vp, int tt, int r) {
  const uint32_t head = vp[tt * D + r];
  const int byte = tt * (D / 2) + (r >> 3) * 4 + (r & 3);
  const uint32_t mb = vp[MID + byte], lb = vp[LOW + byte];
  const bool first = (r & 7) < 4;
  const uint32_t mid = first ? (mb >> 4) : (mb & 0xF);
  const uint32_t low = first ? (lb & 0xF) : (lb >> 4);
  return (head << 8) | (mid << 4) | low;
}

__global__ void __launch_bounds__(ST) select_kernel(akv_store_t s, akv_cfg_t cfg, akv_step_t st, int cap) {
  const int h = blockIdx.x;
  const int G = cfg.group;
  const int u = h / G;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = s.lengths[u];
  const int npg = (n + P - 1) / P;
  __shared__ SelSmem sm;

  // 1. global softmax statistics (fixed assignment + butterfly: deterministic)
  if (warp == 0) {
    const float* ps = st.page_stats + (size_t)h * s.max_pages * 2;
    float m = -INFINITY;
    for (int i = lane; i < npg; i += 32) m = fmaxf(m, ps[2 * i]);
    m = warp_max(m);
    float l = 0.f;
    for (int i = lane; i < npg; i += 32) l += ps[2 * i + 1] * expf(ps[2 * i] - m);
    l = warp_sum(l);
    if (lane == 0) {
      sm.M = m;
      sm.L = l;
    }
  }
  if (tid < 256) sm.hist[tid] = 0;
  __syncthreads();
  const float M = sm.M, L = sm.L;
  const float pmax = 1.0f / L;  // = expf(0) / L, the argmax token's p
  const float thr = ldexpf(pmax, -cfg.m);
  const bool est = cfg.force_tier == 0 && cfg.trunc_bits == 0 && cfg.k_sel > 0;  // k_sel = 0: softmax only
  const float* sc = st.scores + (size_t)h * cap;
  float* pr = st.probs + (size_t)h * cap;

  // 2. probabilities + candidate count
  int ncand = 0;
  for (int t = tid; t < n; t += ST) {
    const float p = expf(sc[t] - M) / L;
    pr[t] = p;
    ncand += (p >= thr);
  }
  ncand = warp_sum_i(ncand);
  if (lane == 0) sm.wcnt[warp][0] = ncand;
  __syncthreads();
  if (tid == 0) {
    int c = 0;
    for (int w = 0; w < ST / 32; ++w) c += sm.wcnt[w][0];
    sm.ncand = c;
    sm.vstar = 0;
    sm.need_eq = 0;
  }
  __syncthreads();
  const int k_sel = max(min(cfg.k_sel, AKV_MAX_KSEL), 1);
  const bool capped = est && sm.ncand > k_sel;

  // 3. radix select of the k_sel-th largest candidate key (only if capped)
  if (capped) {
    unsigned prefix = 0, mask = 0;
    int k = k_sel;
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (int t = tid; t < n; t += ST) {
        const float p = pr[t];
        const unsigned key = __float_as_uint(p);
        if (p >= thr && (key & mask) == prefix) atomicAdd(&sm.hist[(key >> shift) & 0xFF], 1u);
      }
      __syncthreads();
      if (tid == 0) {
        int cum = 0, dg = 255;
        for (; dg > 0; --dg) {
          if (cum + (int)sm.hist[dg] >= k) break;
          cum += sm.hist[dg];
        }
        sm.need_eq = k - cum;  // keys with this digit still needed
        sm.vstar = prefix | ((unsigned)dg << shift);
      }
      __syncthreads();
      k = sm.need_eq;
      prefix = sm.vstar;
      mask |= 0xFFu << shift;
      if (tid < 256) sm.hist[tid] = 0;
      __syncthreads();
    }
  }
  const unsigned vstar = sm.vstar;
  const int need_eq = sm.need_eq;

  // ordered pass: selection flags, bitmap words, ascending index list
  int base_sel = 0, base_eq = 0;
  const int words = (n + 31) >> 5;
  for (int t0 = 0; t0 < n; t0 += ST) {
    const int t = t0 + tid;
    bool cand = false, gt = false, eq = false;
    if (t < n && est) {
      const float p = pr[t];
      cand = p >= thr;
      const unsigned key = __float_as_uint(p);
      gt = cand && key > vstar;
      eq = cand && key == vstar;
    }
    const unsigned beq = __ballot_sync(0xFFFFFFFFu, eq);
    if (lane == 0) sm.wcnt[warp][1] = __popc(beq);
    __syncthreads();
    int eq_before = base_eq;
    for (int w = 0; w < warp; ++w) eq_before += sm.wcnt[w][1];
    eq_before += __popc(beq & ((1u << lane) - 1u));
    const bool sel = capped ? (gt || (eq && eq_before < need_eq)) : cand;
    const unsigned bsel_ = __ballot_sync(0xFFFFFFFFu, sel);
    if (lane == 0 && (t >> 5) < words) st.sel_bits[(size_t)h * (cap >> 5) + (t >> 5)] = bsel_;
    if (lane == 0) sm.wcnt[warp][0] = __popc(bsel_);
    __syncthreads();
    int sel_before = base_sel;
    for (int w = 0; w < warp; ++w) sel_before += sm.wcnt[w][0];
    sel_before += __popc(bsel_ & ((1u << lane) - 1u));
    if (sel && sel_before < AKV_MAX_KSEL) sm.sel_idx[sel_before] = t;
    for (int w = 0; w < ST / 32; ++w) {
      base_sel += sm.wcnt[w][0];
      base_eq += sm.wcnt[w][1];
    }
    __syncthreads();
  }
  const int cnt = min(base_sel, AKV_MAX_KSEL);

  // 4-5. o_est over the selected rows (T16), targets
  if (tid < D) {
    const int r = tid;
    float acc = 0.f;
    for (int i = 0; i < cnt; ++i) {
      const int t = sm.sel_idx[i];
      const uint8_t* vp = page_ptr(s.v_pool, s.page_table, s.max_pages, u, t / P);
      const uint32_t w = v_word_exact(vp, t % P, r);
      acc = fmaf(pr[t], __half2float(__ushort_as_half((unsigned short)w)), acc);
    }
    st.o_est[(size_t)h * D + r] = acc;
    const bool known = acc != 0.f;
    const int tg = known ? floor_log2f(acc) - 10 : AKV_TARGET_UNKNOWN;
    st.targets[(size_t)h * D + r] = tg;
    const int wmin = warp_min_i(known ? tg : INT_MAX);
    const int wunk = warp_sum_i(known ? 0 : 1);
    if (lane == 0) {
      sm.tmin[warp] = wmin;
      sm.tunk[warp] = wunk;
    }
    if (r < cnt) st.sel_idx[(size_t)h * AKV_MAX_KSEL + r] = sm.sel_idx[r];
  }
  __syncthreads();
  if (tid == 0) {
    const int tmin = min(min(sm.tmin[0], sm.tmin[1]), min(sm.tmin[2], sm.tmin[3]));
    const int unk = sm.tunk[0] + sm.tunk[1] + sm.tunk[2] + sm.tunk[3];
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

void launch_select(const akv_store_t& s, const akv_cfg_t& cfg, const akv_step_t& st, cudaStream_t stream) {
  const int cap = s.max_pages * P;
  select_kernel<<<s.n_units * cfg.group, ST, 0, stream>>>(s, cfg, st, cap);
}

}  // namespace akv
