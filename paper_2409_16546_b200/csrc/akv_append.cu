// KVStore.append_token / bulk append: validate, split each
// fp16 word into head byte + two nibbles (HB:154-157), write the paged planes,
// update ColMax and RowMax.
#include "akv_common.cuh"

namespace akv {

// ---------------------------------------------------------------------------
// single-token append: one CTA per unit, thread = channel.
// ---------------------------------------------------------------------------
// pos < 0: append at the unit's length; else truncate the unit to pos tokens (pos <= its
// length) and append there (akv_append_at).
__global__ void __launch_bounds__(D) append_token_kernel(akv_store_t s, const uint16_t* __restrict__ k,
                                                         const uint16_t* __restrict__ v, int64_t* status, int pos) {
  pdl_trigger();
  pdl_wait();
  const int u = blockIdx.x;
  const int c = threadIdx.x;
  // independent loads first (k, v, length), then the page id: two dependent round trips in all
  const uint32_t kw = k[(size_t)u * D + c];
  const uint32_t vw = v[(size_t)u * D + c];
  const int len = s.lengths[u];
  const int t = pos < 0 ? len : pos;
  const bool room = t < s.max_pages * P;
  const size_t pid = room ? (size_t)s.page_table[(size_t)u * s.max_pages + t / P] : 0;
  __shared__ int s_bad;
  __shared__ uint32_t s_rowmax;
  if (c == 0) {
    s_bad = 0x7FFFFFFF;
    s_rowmax = 0;
  }
  __syncthreads();
  // first offending element: K before V, lowest channel (matches the oracle's argwhere order)
  if (!finite16(kw)) atomicMin(&s_bad, c);
  if (!finite16(vw)) atomicMin(&s_bad, 0x100 | c);
  atomicMax(&s_rowmax, vw & 0x7FFFu);
  __syncthreads();
  // status words are sticky: only errors are written, and the first one stays until the
  // caller clears the word (a replayed CUDA graph cannot lose a rejected append)
  if (s_bad != 0x7FFFFFFF) {
    if (c == 0 && status[u] == 0) {
      const int bad = s_bad;
      status[u] = status_word(AKV_STATUS_NONFINITE, ((long long)(bad >> 8) << 59) | ((long long)(bad & 0xFF) << 40));
    }
    return;
  }
  if (!room) {
    if (c == 0 && status[u] == 0) status[u] = status_word(AKV_STATUS_CAPACITY, t);
    return;
  }
  if (t > len) {
    if (c == 0 && status[u] == 0) status[u] = status_word(AKV_STATUS_POSITION, t);
    return;
  }
  const int tt = t % P;
  uint8_t* kp = s.k_pool + pid * PAGE;
  uint8_t* vp = s.v_pool + pid * PAGE;

  // K: channel-major planes.  A nibble word holds 4 token positions of this
  // channel only, so the update is two fire-and-forget reductions (clear, set)
  // instead of a read-modify-write round trip (same-address atomics of one
  // thread are ordered).
  kp[c * P + tt] = (uint8_t)(kw >> 8);
  {
    const int word = (c * (P / 2) + (tt >> 3) * 4) >> 2;
    const bool first = (tt & 7) < 4;
    const int sh = 8 * (tt & 3);
    const int shm = sh + (first ? 4 : 0), shl = sh + (first ? 0 : 4);
    unsigned int* mw = reinterpret_cast<unsigned int*>(kp + MID) + word;
    unsigned int* lw = reinterpret_cast<unsigned int*>(kp + LOW) + word;
    atomicAnd(mw, ~(0xFu << shm));
    atomicOr(mw, ((kw >> 4) & 0xFu) << shm);
    atomicAnd(lw, ~(0xFu << shl));
    atomicOr(lw, (kw & 0xFu) << shl);
  }
  // V: token-major planes; channel c pairs with c+4 inside its 8-group.
  vp[tt * D + c] = (uint8_t)(vw >> 8);
  {
    const uint32_t mn = (vw >> 4) & 0xF, ln = vw & 0xF;
    const uint32_t mn4 = __shfl_down_sync(0xFFFFFFFFu, mn, 4);
    const uint32_t ln4 = __shfl_down_sync(0xFFFFFFFFu, ln, 4);
    if ((c & 7) < 4) {
      const int byte = tt * (D / 2) + (c >> 3) * 4 + (c & 3);
      vp[MID + byte] = (uint8_t)((mn << 4) | mn4);
      vp[LOW + byte] = (uint8_t)(ln | (ln4 << 4));
    }
  }
  // sidecars: ColMax by reduction, RowMax from the block max
  atomicMax(s.colmax + (size_t)u * D + c, kw & 0x7FFFu);
  if (c == 0) {
    s.rowmax[(size_t)u * s.max_pages * P + t] = (uint16_t)s_rowmax;
    s.lengths[u] = t + 1;
  }
}

// ---------------------------------------------------------------------------
// bulk append: validate -> write -> commit.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) append_validate_kernel(akv_store_t s, const uint16_t* __restrict__ k,
                                                              const uint16_t* __restrict__ v, int n_new,
                                                              int64_t* status) {
  const int u = blockIdx.x;
  const size_t base = (size_t)u * n_new * D;
  const long long total = (long long)n_new * D;
  // packed position key: t<<9 | isV<<8 | c  (earliest token, K before V, lowest channel)
  long long best = 0x7FFFFFFFFFFFFFFFLL;
  for (long long i = threadIdx.x; i < total; i += blockDim.x) {
    const uint32_t kw = k[base + i], vw = v[base + i];
    const long long t = i / D, c = i % D;
    if (!finite16(kw)) best = min(best, (t << 9) | c);
    if (!finite16(vw)) best = min(best, (t << 9) | 0x100 | c);
  }
  __shared__ long long s_best[8];
#pragma unroll
  for (int o = 16; o; o >>= 1) best = min(best, __shfl_xor_sync(0xFFFFFFFFu, best, o));
  if ((threadIdx.x & 31) == 0) s_best[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) best = min(best, s_best[w]);
    const int t0 = s.lengths[u];
    if (status[u] != 0) {
      // an earlier rejection is still pending (sticky): this append is refused too
    } else if (best != 0x7FFFFFFFFFFFFFFFLL) {
      const long long t = best >> 9, isv = (best >> 8) & 1, c = best & 0xFF;
      status[u] = status_word(AKV_STATUS_NONFINITE, (isv << 59) | (c << 40) | t);
    } else if ((long long)t0 + n_new > (long long)s.max_pages * P) {
      status[u] = status_word(AKV_STATUS_CAPACITY, t0);
    }
  }
}

// grid (chunks, U); chunk = one page-aligned span of P positions.
__global__ void __launch_bounds__(256) append_bulk_kernel(akv_store_t s, const uint16_t* __restrict__ k,
                                                          const uint16_t* __restrict__ v, int n_new,
                                                          const int64_t* __restrict__ status) {
  const int u = blockIdx.y;
  if (status[u] != 0) return;
  const int t0 = s.lengths[u];
  // positions [t0, t0+n_new) split at page boundaries; chunk j covers page (t0/P + j)
  const int pg = t0 / P + blockIdx.x;
  const int lo = max(t0, pg * P), hi = min(t0 + n_new, (pg + 1) * P);
  if (lo >= hi) return;
  uint8_t* kp = s.k_pool + (size_t)s.page_table[(size_t)u * s.max_pages + pg] * PAGE;
  uint8_t* vp = s.v_pool + (size_t)s.page_table[(size_t)u * s.max_pages + pg] * PAGE;
  const uint16_t* kin = k + (size_t)u * n_new * D;
  const uint16_t* vin = v + (size_t)u * n_new * D;
  const int ntok = hi - lo;
  // heads + rowmax: thread per (token, channel)
  for (int i = threadIdx.x; i < ntok * D; i += blockDim.x) {
    const int tt = lo + i / D - pg * P, c = i % D;
    const size_t src = (size_t)(lo - t0 + i / D) * D + c;
    kp[c * P + tt] = (uint8_t)(kin[src] >> 8);
    vp[tt * D + c] = (uint8_t)(vin[src] >> 8);
  }
  // rowmax: warp per token
  for (int r = threadIdx.x >> 5; r < ntok; r += blockDim.x >> 5) {
    const size_t src = (size_t)(lo - t0 + r) * D;
    uint32_t m = 0;
    for (int c = threadIdx.x & 31; c < D; c += 32) m = max(m, (uint32_t)vin[src + c] & 0x7FFFu);
#pragma unroll
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
    if ((threadIdx.x & 31) == 0) s.rowmax[(size_t)u * s.max_pages * P + lo + r] = (uint16_t)m;
  }
  // K nibble words: thread per (channel, 8-token group); RMW partial groups
  const int g_lo = (lo - pg * P) >> 3, g_hi = (hi - pg * P + 7) >> 3;
  for (int i = threadIdx.x; i < D * (g_hi - g_lo); i += blockDim.x) {
    const int c = i % D, g = g_lo + i / D;
    uint32_t* mw = reinterpret_cast<uint32_t*>(kp + MID + c * (P / 2) + g * 4);
    uint32_t* lw = reinterpret_cast<uint32_t*>(kp + LOW + c * (P / 2) + g * 4);
    uint32_t m = *mw, l = *lw;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int tt = g * 8 + e, t = pg * P + tt;
      if (t < lo || t >= hi) continue;
      const uint32_t w = kin[(size_t)(t - t0) * D + c];
      const uint32_t mn = (w >> 4) & 0xF, ln = w & 0xF;
      const int byte = e & 3;
      if (e < 4) {
        m = (m & ~(0xF0u << (8 * byte))) | (mn << (8 * byte + 4));
        l = (l & ~(0x0Fu << (8 * byte))) | (ln << (8 * byte));
      } else {
        m = (m & ~(0x0Fu << (8 * byte))) | (mn << (8 * byte));
        l = (l & ~(0xF0u << (8 * byte))) | (ln << (8 * byte + 4));
      }
    }
    *mw = m;
    *lw = l;
  }
  // V nibble words: thread per (token, 8-channel group); whole words
  for (int i = threadIdx.x; i < ntok * (D / 8); i += blockDim.x) {
    const int r = i / (D / 8), g = i % (D / 8);
    const int tt = lo + r - pg * P;
    const uint16_t* src = vin + (size_t)(lo - t0 + r) * D + g * 8;
    uint32_t m = 0, l = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t a = src[e], b = src[e + 4];
      m |= ((((a >> 4) & 0xF) << 4) | ((b >> 4) & 0xF)) << (8 * e);
      l |= ((a & 0xF) | ((b & 0xF) << 4)) << (8 * e);
    }
    *reinterpret_cast<uint32_t*>(vp + MID + tt * (D / 2) + g * 4) = m;
    *reinterpret_cast<uint32_t*>(vp + LOW + tt * (D / 2) + g * 4) = l;
  }
  // colmax: thread per channel over this chunk's tokens
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    uint32_t m = 0;
    for (int t = lo; t < hi; ++t) m = max(m, (uint32_t)kin[(size_t)(t - t0) * D + c] & 0x7FFFu);
    atomicMax(s.colmax + (size_t)u * D + c, m);
  }
}

__global__ void append_commit_kernel(akv_store_t s, int n_new, const int64_t* __restrict__ status) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u < s.n_units && status[u] == 0) s.lengths[u] += n_new;
}

// ---------------------------------------------------------------------------
// Prefill writer (bulk append with a caller workspace): one CTA per (unit, half page
// span of 128 positions), validation fused in, ColMax and the commit deferred to a
// per-unit kernel.  No shared memory: the K transpose goes through registers.
//
// K (channel-major page): warp w owns channel pairs 32 (w & 1) + lane and the 32
// positions 32 (w >> 1) .. of the half page; lane loads its pair's 32 words as 32 4 B
// loads, each warp load being one coalesced 128 B segment of a token row, then stores
// per channel 2 x 16 B of head bytes and 16 B of each nibble plane (the 8-token nibble
// words of akv.h).  V (token-major, like the input): thread = (token, 8 channels), one
// 16 B load, an 8 B head store and a 4 B store per nibble word, RowMax by a 16-lane max.
// Only the 16-position groups cut by the span ends merge with the page's bytes.
// Non-finite words: the earliest (token, K before V, channel) key, atomicMin into the
// unit's workspace key; ColMax: atomicMax into the unit's workspace row (both reset by
// akv_append_ws).  akv_append_commit_ws_kernel rejects the unit's whole append on any
// key (D10) or folds the ColMax row and bumps the length; planes / RowMax beyond the
// length are never read, so a rejected append leaves nothing visible.
// ---------------------------------------------------------------------------
constexpr int PF_THREADS = 256;

__device__ __forceinline__ uint32_t nonfinite_mask2(uint32_t w) {
  // bit 15 / 31 set where the half's exponent field is all ones (t + 0x400 carries into bit 15)
  return ((w & 0x7C007C00u) + 0x04000400u) & 0x80008000u;
}

// 16 positions x a channel pair (w[e] = channel 2cp+1 word << 16 | channel 2cp word):
// per channel the 16 head bytes (4 words) and the two 8-position mid / low nibble words
// (akv.h packing: mid byte i = mid(i) << 4 | mid(i + 4), low byte i = low(i) | low(i + 4) << 4).
// Byte gathers by PRMT, nibble words by two LOP3 + shift each.
__device__ __forceinline__ void pack16x2(const uint32_t* w, uint32_t (&h)[2][4], uint32_t (&m)[2][2],
                                         uint32_t (&l)[2][2]) {
  uint32_t lb[2][4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t a = prmt(w[4 * q], w[4 * q + 1], 0x7351), b = prmt(w[4 * q + 2], w[4 * q + 3], 0x7351);
    h[0][q] = prmt(a, b, 0x5410);
    h[1][q] = prmt(a, b, 0x7632);
    const uint32_t c = prmt(w[4 * q], w[4 * q + 1], 0x6240), d = prmt(w[4 * q + 2], w[4 * q + 3], 0x6240);
    lb[0][q] = prmt(c, d, 0x5410);
    lb[1][q] = prmt(c, d, 0x7632);
  }
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int wi = 0; wi < 2; ++wi) {
      const uint32_t A = lb[j][2 * wi], B = lb[j][2 * wi + 1];
      m[j][wi] = bsel(0xF0F0F0F0u, A, B >> 4);
      l[j][wi] = bsel(0x0F0F0F0Fu, A, B << 4);
    }
}

__device__ __forceinline__ void store16(uint8_t* kp, int c, int tg0, uint32_t cover, const uint32_t (&h)[4],
                                        const uint32_t (&m)[2], const uint32_t (&l)[2]) {
  uint4* hd = reinterpret_cast<uint4*>(kp + c * P + tg0);
  uint2* md = reinterpret_cast<uint2*>(kp + MID + c * (P / 2) + tg0 / 2);
  uint2* ld = reinterpret_cast<uint2*>(kp + LOW + c * (P / 2) + tg0 / 2);
  if (cover == 0xFFFFu) {
    *hd = make_uint4(h[0], h[1], h[2], h[3]);
    *md = make_uint2(m[0], m[1]);
    *ld = make_uint2(l[0], l[1]);
    return;
  }
  // a group cut by the span ends: keep the page's bytes / nibbles of the other positions
  const uint4 oh = *hd;
  const uint2 om = *md, ol = *ld;
  uint32_t hm[4], nm[2], nl[2];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t mk = 0u;
#pragma unroll
    for (int b = 0; b < 4; ++b) mk |= ((cover >> (4 * q + b)) & 1u) ? (0xFFu << (8 * b)) : 0u;
    hm[q] = mk;
  }
#pragma unroll
  for (int wi = 0; wi < 2; ++wi) {
    uint32_t mm = 0u, lm = 0u;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      if (!((cover >> (8 * wi + e)) & 1u)) continue;
      const int by = e & 3;
      mm |= (e < 4 ? 0xF0u : 0x0Fu) << (8 * by);
      lm |= (e < 4 ? 0x0Fu : 0xF0u) << (8 * by);
    }
    nm[wi] = mm;
    nl[wi] = lm;
  }
  *hd = make_uint4(bsel(hm[0], h[0], oh.x), bsel(hm[1], h[1], oh.y), bsel(hm[2], h[2], oh.z), bsel(hm[3], h[3], oh.w));
  *md = make_uint2(bsel(nm[0], m[0], om.x), bsel(nm[1], m[1], om.y));
  *ld = make_uint2(bsel(nl[0], l[0], ol.x), bsel(nl[1], l[1], ol.y));
}

__global__ void __launch_bounds__(PF_THREADS) append_page_kernel(akv_store_t s, const uint16_t* __restrict__ k,
                                                                 const uint16_t* __restrict__ v, int n_new,
                                                                 const int64_t* __restrict__ status,
                                                                 uint32_t* __restrict__ ws_colmax,
                                                                 unsigned long long* __restrict__ ws_bad) {
  const int u = blockIdx.y, hs = blockIdx.x & 1, ch = blockIdx.x >> 1, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int t0 = s.lengths[u];
  const int pg = t0 / P + ch;
  const int base = pg * P + hs * (P / 2);  // first position of this half page
  const int lo = max(t0, base), hi = min(t0 + n_new, base + P / 2);
  // refused (sticky status), beyond capacity (the commit reports it) or an empty span
  if (status[u] != 0 || (long long)t0 + n_new > (long long)s.max_pages * P || lo >= hi) return;
  const size_t pid = (size_t)s.page_table[(size_t)u * s.max_pages + pg];
  uint8_t* kp = s.k_pool + pid * PAGE;
  uint8_t* vp = s.v_pool + pid * PAGE;
  const uint16_t* kin = k + (size_t)u * n_new * D;
  const uint16_t* vin = v + (size_t)u * n_new * D;
  unsigned long long bad = ~0ull;

  // K: channel pair cp, positions base + 32 (warp >> 1) .. + 31
  {
    const int cp = 32 * (warp & 1) + lane;
    const int p0 = base + 32 * (warp >> 1);
    uint32_t w2[32];
    uint32_t cover = 0u;
#pragma unroll
    for (int e = 0; e < 32; ++e) {
      const int t = p0 + e;
      const bool in = t >= lo && t < hi;
      cover |= (in ? 1u : 0u) << e;
      w2[e] = in ? *reinterpret_cast<const uint32_t*>(kin + (size_t)(t - t0) * D + 2 * cp) : 0u;
    }
    if (cover) {
      uint32_t cm = 0u, nf = 0u;
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        nf |= nonfinite_mask2(w2[e]);
        cm = __vmaxu2(cm, w2[e] & 0x7FFF7FFFu);
      }
      if (nf) {  // rare: the exact earliest position (words reloaded: no indexed register array)
#pragma unroll 1
        for (int e = 0; e < 32; ++e) {
          if (!((cover >> e) & 1u)) continue;
          const uint32_t x = *reinterpret_cast<const uint32_t*>(kin + (size_t)(p0 + e - t0) * D + 2 * cp);
#pragma unroll
          for (int j = 0; j < 2; ++j)
            if (!finite16((x >> (16 * j)) & 0xFFFFu))
              bad = min(bad, ((unsigned long long)(p0 + e - t0) << 9) | (unsigned long long)(2 * cp + j));
        }
      }
      atomicMax(ws_colmax + (size_t)u * D + 2 * cp, cm & 0xFFFFu);
      atomicMax(ws_colmax + (size_t)u * D + 2 * cp + 1, cm >> 16);
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const uint32_t cv = (cover >> (16 * half)) & 0xFFFFu;
        if (!cv) continue;
        uint32_t h[2][4], m[2][2], l[2][2];
        pack16x2(w2 + 16 * half, h, m, l);
#pragma unroll
        for (int j = 0; j < 2; ++j) store16(kp, 2 * cp + j, p0 + 16 * half - pg * P, cv, h[j], m[j], l[j]);
      }
    }
  }
  // V: thread = (position, 8 channels), 8 items per thread with every load issued first;
  // RowMax over the 16 threads of a position
  constexpr int VI = (P / 2) * 16 / PF_THREADS;
  uint4 vw[VI];
#pragma unroll
  for (int k = 0; k < VI; ++k) {
    const int i = tid + k * PF_THREADS, t = base + (i >> 4);
    vw[k] = (t >= lo && t < hi) ? *reinterpret_cast<const uint4*>(vin + (size_t)(t - t0) * D + 8 * (i & 15))
                                : make_uint4(0u, 0u, 0u, 0u);
  }
#pragma unroll
  for (int k = 0; k < VI; ++k) {
    const int i = tid + k * PF_THREADS, r = i >> 4, g = i & 15;
    const int t = base + r;
    const bool in = t >= lo && t < hi;
    const uint4 w = vw[k];
    uint32_t m = 0u;
    if (in) {
      if (nonfinite_mask2(w.x) | nonfinite_mask2(w.y) | nonfinite_mask2(w.z) | nonfinite_mask2(w.w)) {
        const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (!finite16((wv[e >> 1] >> (16 * (e & 1))) & 0xFFFFu))
            bad = min(bad, ((unsigned long long)(t - t0) << 9) | 0x100ull | (unsigned long long)(8 * g + e));
      }
      // head bytes (byte 1 of each word), low bytes (byte 0), nibble words of the 8-channel
      // group (channel c pairs with c + 4, akv.h)
      const uint32_t hb0 = prmt(w.x, w.y, 0x7531), hb1 = prmt(w.z, w.w, 0x7531);
      const uint32_t A = prmt(w.x, w.y, 0x6420), B = prmt(w.z, w.w, 0x6420);
      const uint32_t mw = bsel(0xF0F0F0F0u, A, B >> 4), lw = bsel(0x0F0F0F0Fu, A, B << 4);
      const uint32_t mx = __vmaxu2(__vmaxu2(w.x & 0x7FFF7FFFu, w.y & 0x7FFF7FFFu),
                                   __vmaxu2(w.z & 0x7FFF7FFFu, w.w & 0x7FFF7FFFu));
      m = max(mx & 0xFFFFu, mx >> 16);
      const int tt = t - pg * P;
      *reinterpret_cast<uint2*>(vp + tt * D + 8 * g) = make_uint2(hb0, hb1);
      *reinterpret_cast<uint32_t*>(vp + MID + tt * (D / 2) + 4 * g) = mw;
      *reinterpret_cast<uint32_t*>(vp + LOW + tt * (D / 2) + 4 * g) = lw;
    }
#pragma unroll
    for (int o = 8; o; o >>= 1) m = max(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
    if (in && g == 0) s.rowmax[(size_t)u * s.max_pages * P + t] = (uint16_t)m;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const unsigned long long y = __shfl_xor_sync(0xFFFFFFFFu, bad, o);
    bad = min(bad, y);
  }
  if (lane == 0 && bad != ~0ull) atomicMin(ws_bad + u, bad);
}

// Per unit: reject (sticky status: capacity, or the earliest non-finite word) or commit
// (ColMax row folded in, length += n_new).
__global__ void __launch_bounds__(D) append_commit_ws_kernel(akv_store_t s, int n_new, int64_t* status,
                                                             const uint32_t* __restrict__ ws_colmax,
                                                             const unsigned long long* __restrict__ ws_bad) {
  const int u = blockIdx.x, c = threadIdx.x;
  if (status[u] != 0) return;  // an earlier rejection is pending: this append was refused
  const int t0 = s.lengths[u];
  if ((long long)t0 + n_new > (long long)s.max_pages * P) {
    if (c == 0) status[u] = status_word(AKV_STATUS_CAPACITY, t0);
    return;
  }
  const unsigned long long bad = ws_bad[u];
  if (bad != ~0ull) {
    if (c == 0) {
      const long long t = (long long)(bad >> 9), isv = (long long)((bad >> 8) & 1), cc = (long long)(bad & 0xFF);
      status[u] = status_word(AKV_STATUS_NONFINITE, (isv << 59) | (cc << 40) | t);
    }
    return;
  }
  atomicMax(s.colmax + (size_t)u * D + c, ws_colmax[(size_t)u * D + c]);
  __syncthreads();
  if (c == 0) s.lengths[u] = t0 + n_new;
}

// ---------------------------------------------------------------------------
// Metered reads (KVStore.read_element / read_channel): one thread per
// request reads only the planes its tier needs (head byte; + mid nibble for T12 / T16;
// + low nibble for T16), rebuilds the word with the midpoint fill (HB:160-179) and
// counts the element at its tier (warp-aggregated atomics); SKIP reads nothing and
// returns 0.  Out-of-range requests return 0 and are not counted.
// ---------------------------------------------------------------------------
__global__ void read_elements_kernel(akv_store_t s, int which, const int32_t* __restrict__ unit,
                                     const int32_t* __restrict__ tok, const int32_t* __restrict__ chan,
                                     const int32_t* __restrict__ tier, long long n, uint16_t* __restrict__ out,
                                     unsigned long long* __restrict__ counters) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  int code = 0;
  uint32_t w = 0u;
  if (i < n) {
    const int u = unit[i], t = tok[i], c = chan[i];
    code = tier[i];
    if (u < 0 || u >= s.n_units || c < 0 || c >= D || t < 0 || t >= s.lengths[u] || code == 0) {
      code = 0;
    } else {
      const uint8_t* pg = (which ? s.v_pool : s.k_pool) +
                          (size_t)s.page_table[(size_t)u * s.max_pages + t / P] * PAGE;
      const int tt = t % P;
      int hb, nb;
      bool hi;  // mid nibble in the high half of its byte (low nibble in the other half)
      if (which == 0) {  // K: channel-major, nibble words over 8 tokens
        hb = c * P + tt;
        nb = c * (P / 2) + (tt >> 3) * 4 + (tt & 3);
        hi = (tt & 7) < 4;
      } else {  // V: token-major, nibble words over 8 channels
        hb = tt * D + c;
        nb = tt * (D / 2) + (c >> 3) * 4 + (c & 3);
        hi = (c & 7) < 4;
      }
      w = (uint32_t)pg[hb] << 8;
      if (code >= 12) {
        const uint32_t mb = pg[MID + nb];
        w |= (hi ? (mb >> 4) : (mb & 0xFu)) << 4;
        if (code >= 16) {
          const uint32_t lb = pg[LOW + nb];
          w |= hi ? (lb & 0xFu) : (lb >> 4);
        } else {
          w |= 0x8u;
        }
      } else {
        w |= 0x80u;
      }
    }
    out[i] = (uint16_t)w;
  }
  const unsigned lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const unsigned b = __ballot_sync(0xFFFFFFFFu, code == 8 + 4 * k);
    if (b && lane == 0) atomicAdd(counters + k, (unsigned long long)__popc(b));
  }
}

}  // namespace akv

using namespace akv;

extern "C" int akv_read_elements(const akv_store_t* store, int32_t which, const int32_t* unit, const int32_t* tok,
                                 const int32_t* chan, const int32_t* tier, int64_t n, uint16_t* out, int64_t* counters,
                                 void* stream) {
  if (!store || (which != 0 && which != 1) || n < 0 || (n > 0 && (!unit || !tok || !chan || !tier || !out)) ||
      !counters)
    return AKV_EINVAL;
  if (store->head_dim != D) return AKV_EUNSUPPORTED;
  if (n == 0) return AKV_OK;
  const int threads = 256;
  read_elements_kernel<<<(unsigned)((n + threads - 1) / threads), threads, 0, (cudaStream_t)stream>>>(
      *store, which, unit, tok, chan, tier, n, out, reinterpret_cast<unsigned long long*>(counters));
  return cudaGetLastError() == cudaSuccess ? AKV_OK : AKV_ECUDA;
}

extern "C" int64_t akv_append_workspace_bytes(int32_t n_units, int32_t n_new) {
  if (n_units <= 0 || n_new <= 0) return 0;
  return (long long)n_units * (D * 4 + 8);  // ColMax row + earliest non-finite key per unit
}

extern "C" int akv_append_ws(const akv_store_t* store, const uint16_t* k, const uint16_t* v, int32_t n_new,
                             int64_t* status, void* workspace, int64_t workspace_bytes, void* stream) {
  if (!store || !k || !v || !status || n_new < 0) return AKV_EINVAL;
  if (store->head_dim != D) return AKV_EUNSUPPORTED;
  if (n_new == 0 || store->n_units == 0) return AKV_OK;
  if (n_new == 1) return akv_append(store, k, v, n_new, status, stream);
  if (!workspace || workspace_bytes < akv_append_workspace_bytes(store->n_units, n_new)) return AKV_EINVAL;
  if ((reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v)) & 15) return AKV_EINVAL;  // 16 B loads
  cudaStream_t st = (cudaStream_t)stream;
  const int chunks = (n_new + P - 1) / P + 1;  // page spans (the first may start mid-page)
  uint32_t* ws_colmax = reinterpret_cast<uint32_t*>(workspace);
  unsigned long long* ws_bad = reinterpret_cast<unsigned long long*>(ws_colmax + (size_t)store->n_units * D);
  cudaMemsetAsync(ws_colmax, 0, (size_t)store->n_units * D * 4, st);
  cudaMemsetAsync(ws_bad, 0xFF, (size_t)store->n_units * 8, st);
  append_page_kernel<<<dim3(2 * chunks, store->n_units), PF_THREADS, 0, st>>>(*store, k, v, n_new, status, ws_colmax,
                                                                            ws_bad);
  append_commit_ws_kernel<<<store->n_units, D, 0, st>>>(*store, n_new, status, ws_colmax, ws_bad);
  return cudaGetLastError() == cudaSuccess ? AKV_OK : AKV_ECUDA;
}

extern "C" int akv_append(const akv_store_t* store, const uint16_t* k, const uint16_t* v, int32_t n_new,
                          int64_t* status, void* stream) {
  if (!store || !k || !v || !status || n_new < 0) return AKV_EINVAL;
  if (store->head_dim != D) return AKV_EUNSUPPORTED;
  if (n_new == 0 || store->n_units == 0) return AKV_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (n_new == 1) {
    launch_pdl(PDL_APPEND, append_token_kernel, dim3(store->n_units), dim3(D), 0, st, *store, k, v, status, -1);
  } else {
    append_validate_kernel<<<store->n_units, 256, 0, st>>>(*store, k, v, n_new, status);
    const int chunks = (n_new + P - 1) / P + 1;
    append_bulk_kernel<<<dim3(chunks, store->n_units), 256, 0, st>>>(*store, k, v, n_new, status);
    append_commit_kernel<<<(store->n_units + 127) / 128, 128, 0, st>>>(*store, n_new, status);
  }
  return cudaGetLastError() == cudaSuccess ? AKV_OK : AKV_ECUDA;
}

extern "C" int akv_append_at(const akv_store_t* store, const uint16_t* k, const uint16_t* v, int32_t pos,
                             int64_t* status, void* stream) {
  if (!store || !k || !v || !status || pos < 0) return AKV_EINVAL;
  if (store->head_dim != D) return AKV_EUNSUPPORTED;
  if (store->n_units == 0) return AKV_OK;
  launch_pdl(PDL_APPEND, append_token_kernel, dim3(store->n_units), dim3(D), 0, (cudaStream_t)stream, *store, k, v,
             status, pos);
  return cudaGetLastError() == cudaSuccess ? AKV_OK : AKV_ECUDA;
}
