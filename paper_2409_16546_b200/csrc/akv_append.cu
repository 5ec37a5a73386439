// KVStore.append_token / bulk append: validate, split each
// fp16 word into head byte + two nibbles (HB:154-157), write the paged planes,
// update ColMax and RowMax.
#include "akv_common.cuh"

namespace akv {

// ---------------------------------------------------------------------------
// single-token append: one CTA per unit, thread = channel.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(D) append_token_kernel(akv_store_t s, const uint16_t* __restrict__ k,
                                                         const uint16_t* __restrict__ v, int64_t* status) {
  pdl_trigger();
  pdl_wait();
  const int u = blockIdx.x;
  const int c = threadIdx.x;
  // independent loads first (k, v, length), then the page id: two dependent round trips in all
  const uint32_t kw = k[(size_t)u * D + c];
  const uint32_t vw = v[(size_t)u * D + c];
  const int t = s.lengths[u];
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

}  // namespace akv

using namespace akv;

extern "C" int akv_append(const akv_store_t* store, const uint16_t* k, const uint16_t* v, int32_t n_new,
                          int64_t* status, void* stream) {
  if (!store || !k || !v || !status || n_new < 0) return AKV_EINVAL;
  if (store->head_dim != D) return AKV_EUNSUPPORTED;
  if (n_new == 0 || store->n_units == 0) return AKV_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (n_new == 1) {
    launch_pdl(append_token_kernel, dim3(store->n_units), dim3(D), 0, st, *store, k, v, status);
  } else {
    append_validate_kernel<<<store->n_units, 256, 0, st>>>(*store, k, v, n_new, status);
    const int chunks = (n_new + P - 1) / P + 1;
    append_bulk_kernel<<<dim3(chunks, store->n_units), 256, 0, st>>>(*store, k, v, n_new, status);
    append_commit_kernel<<<(store->n_units + 127) / 128, 128, 0, st>>>(*store, n_new, status);
  }
  return cudaGetLastError() == cudaSuccess ? AKV_OK : AKV_ECUDA;
}
