// Shared device helpers for the libakv kernels (sm_100a).
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#include "akv.h"


namespace akv {

constexpr int D = AKV_HEAD_DIM;
constexpr int P = AKV_PAGE_TOKENS;
constexpr int PAGE = AKV_PAGE_BYTES;
constexpr int MID = AKV_PAGE_MID_OFF;
constexpr int LOW = AKV_PAGE_LOW_OFF;

// fp16 pattern helpers -------------------------------------------------------
__device__ __forceinline__ int bexp16(uint32_t w) { return (w >> 10) & 0x1F; }
__device__ __forceinline__ bool finite16(uint32_t w) { return (w & 0x7C00u) != 0x7C00u; }

// floor(log2|x|) of a finite non-zero fp16 pattern (HB:108-118, subnormal aware).
__device__ __forceinline__ int magexp16(uint32_t w) {
  const int b = bexp16(w);
  if (b) return b - 15;
  const uint32_t m = w & 0x3FFu;  // caller guarantees m != 0
  return (31 - __clz(m)) - 24;
}

// floor(log2|x|) of a finite non-zero fp32 value (frexp exponent - 1).
__device__ __forceinline__ int floor_log2f(float x) {
  const uint32_t b = __float_as_uint(x) & 0x7FFFFFFFu;
  const int e = (int)(b >> 23);
  if (e) return e - 127;
  return (31 - __clz(b)) - 149;
}

// Byte permute (PRMT).
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

// Bit select: (a & m) | (b & ~m)  — a single LOP3.
__device__ __forceinline__ uint32_t bsel(uint32_t m, uint32_t a, uint32_t b) { return (a & m) | (b & ~m); }

// Assemble the 8 fp16 words of one 8-group from its head bytes (h0: elements
// 0..3, h1: 4..7) and the group's mid / low words (packing in akv.h).
// out[k] holds elements (2k, 2k+1) as a half2 bit pattern.
__device__ __forceinline__ void assemble8(uint32_t h0, uint32_t h1, uint32_t mid, uint32_t low, uint32_t out[4]) {
  const uint32_t x = bsel(0xF0F0F0F0u, mid, low);              // low bytes of elements 0..3
  const uint32_t y = bsel(0xF0F0F0F0u, mid << 4, low >> 4);    // low bytes of elements 4..7
  out[0] = prmt(x, h0, 0x5140);
  out[1] = prmt(x, h0, 0x7362);
  out[2] = prmt(y, h1, 0x5140);
  out[3] = prmt(y, h1, 0x7362);
}

// Tier masks: mid' = bsel(mk, mid, 0x88888888); low' = bsel(lk, low, lf).
struct TierMask {
  uint32_t mk, lk, lf;
};
__device__ __forceinline__ TierMask tier_mask(int code) {
  TierMask t;
  t.mk = code >= 12 ? 0xFFFFFFFFu : 0u;
  t.lk = code >= 16 ? 0xFFFFFFFFu : 0u;
  t.lf = code == 12 ? 0x88888888u : 0u;
  return t;
}

// Streaming global loads: read-only, no L1 allocation, L2 evict-first policy
// (the KV planes are read once per step; keep L2 for scores / probs).
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint2 ld_stream_u64(const void* p, uint64_t pol) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
               : "=r"(r.x), "=r"(r.y)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ uint4 ld_stream_u128(const void* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

// ---------------------------------------------------------------------------
// mbarrier + TMA bulk copy (cp.async.bulk, SASS UBLKCP) helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// One elected lane of a converged warp (elect.sync): warp-uniform operands of the elected
// lane's TMA / MMA issue stay in uniform registers (no per-lane R2UR waterfall).
__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(p));
  return p != 0;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Watchdog: a protocol bug must fail the launch (trap -> cudaErrorLaunchFailure),
// never hang the GPU: a wait longer than 2 s of wall time traps.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  const uint64_t t0 = globaltimer_ns();
  uint32_t spins = 0;
  while (!mbar_try_wait(bar, parity)) {
    if ((++spins & 1023u) == 0 && globaltimer_ns() - t0 > 2000000000ull) __trap();
  }
}
// Bulk global -> shared copy completing on an mbarrier (bytes % 16 == 0, 16 B aligned).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// 16-byte cp.async (LDGSTS, L2 only).
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}


__device__ __forceinline__ float2 half2_bits_to_float2(uint32_t w) {
  __half2 h = *reinterpret_cast<__half2*>(&w);
  return __half22float2(h);
}

// acc(x,y) += p * (v.x, v.y) via the packed FFMA2.
__device__ __forceinline__ float2 ffma2_scalar(float2 v, float p, float2 acc) {
  float2 r;
  const float2 pp = make_float2(p, p);
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&r))
      : "l"(*reinterpret_cast<const unsigned long long*>(&v)),
        "l"(*reinterpret_cast<const unsigned long long*>(&pp)),
        "l"(*reinterpret_cast<const unsigned long long*>(&acc)));
  return r;
}

// Warp reductions.
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}
__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}
__device__ __forceinline__ int warp_max_i(int v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
  return v;
}
__device__ __forceinline__ int warp_min_i(int v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
  return v;
}

// A unit's page-table row held in the producer warp's registers: lane l keeps
// the pool ids of pages l, l+32, l+64, l+96 (contexts up to 32k tokens; longer
// ones fall back to a global load).  Loaded one unit ahead so the producers
// never wait on a dependent global load between stages.
struct UnitPages {
  int u, n;
  int pt[4];
};
__device__ __forceinline__ void unit_pages_fetch(UnitPages& f, const akv_store_t& s, int u) {
  const int lane = threadIdx.x & 31;
  f.u = u;
  f.n = s.lengths[u];
  const int32_t* row = s.page_table + (size_t)u * s.max_pages;
#pragma unroll
  for (int k = 0; k < 4; ++k) f.pt[k] = lane + 32 * k < s.max_pages ? row[lane + 32 * k] : 0;
}
__device__ __forceinline__ size_t unit_page(const UnitPages& f, const akv_store_t& s, int pg) {
  const int k = pg >> 5;  // warp-uniform
  int v = k == 0 ? f.pt[0] : (k == 1 ? f.pt[1] : (k == 2 ? f.pt[2] : f.pt[3]));
  v = __shfl_sync(0xFFFFFFFFu, v, pg & 31);
  if (pg >= 128) v = s.page_table[(size_t)f.u * s.max_pages + pg];
  return (size_t)v;
}

// Programmatic dependent launch (PDL): every step kernel is launched with
// programmatic stream serialization, lets its dependent start launching at
// once, and waits for its predecessor's memory before touching any of it, so
// launch latency overlaps the previous kernel's tail.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Kernel classes of the decode chain.  AKV_NOPDL (bit mask of classes, A/B probes) launches
// those classes without programmatic stream serialization.
enum { PDL_APPEND = 0, PDL_QK = 1, PDL_SELECT = 2, PDL_PV = 3, PDL_COMBINE = 4, PDL_OFF = 30 };
inline int env_int(const char* name, int dflt);
inline int nopdl_mask() {
  static const int m = env_int("AKV_NOPDL", 1 << PDL_APPEND);
  return m;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(int cls, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t lc = {};
  lc.gridDim = grid;
  lc.blockDim = block;
  lc.dynamicSmemBytes = smem;
  lc.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = (cls == PDL_OFF || ((nopdl_mask() >> cls) & 1)) ? 0 : 1;
  return cudaLaunchKernelEx(&lc, kernel, args...);
}

// Resident CTAs of a kernel across the current device (SMs x occupancy), with the
// dynamic shared-memory opt-in applied.  Both are per-device properties, so the
// cache is keyed by the device ordinal (one process may drive several GPUs);
// computing an entry twice under a race is harmless (idempotent).
constexpr int MAX_DEVICES = 64;
template <auto Kern>
inline int resident_ctas(int threads, size_t smem) {
  static int cache[MAX_DEVICES] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int* slot = dev >= 0 && dev < MAX_DEVICES ? &cache[dev] : nullptr;
  if (slot && *slot) return *slot;
  int sms = 0, per = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (smem > 48 * 1024) cudaFuncSetAttribute(Kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, Kern, threads, smem);
  const int r = sms * (per > 0 ? per : 1);
  if (slot) *slot = r;
  return r;
}

// Host: CTAs of `warps` warps for a static split of `items` warp-items (contiguous balanced
// ranges) when `resident` CTAs fit the device: the fewest CTAs that keep the per-warp
// maximum at ceil(items / resident warps).  With 4.6 items per resident warp, every warp
// otherwise ends at 4 or 5 items and the 4-item warps idle through the last round; with
// the trimmed grid (nearly) every warp runs 5 and the kernel's bytes are spread over
// slightly fewer warps.  AKV_GRID_BALANCE=0 keeps the full resident grid (A/B).
inline int env_int(const char* name, int dflt);
inline int balanced_grid(long long items, int resident, int warps, bool allow = true) {
  static const int on = env_int("AKV_GRID_BALANCE", 1);
  const long long full = std::max<long long>(std::min<long long>(resident, (items + warps - 1) / warps), 1);
  if (!on || !allow) return (int)full;
  const long long rw = (long long)resident * warps;
  const long long k = std::max<long long>((items + rw - 1) / rw, 1);  // items per warp at most
  // trim only when the last round leaves >= 5 % of the warp-time idle (measured: c2 4.61 items
  // per warp, 147.0 -> 143.8 us; c4 18.45 items per warp: trimming costs more bytes in flight
  // than the 3 % tail it removes)
  if (20 * (k * rw - items) < k * rw) return (int)full;
  const long long w = (items + k - 1) / k;                           // warps needed for that
  return (int)std::max<long long>(std::min<long long>((w + warps - 1) / warps, full), 1);
}

// Host: integer knob from the environment (A/B measurements), read once by the caller.
inline int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e && *e ? atoi(e) : dflt;
}

// Host: row-major 2-D tensor map (TMA) over a device buffer, cached per (base, shape, box,
// swizzle) and thread.  The driver entry point is fetched through the runtime (no -lcuda).
inline bool tmap_2d(void* base, CUtensorMapDataType dt, int esize, unsigned long long inner, unsigned long long outer,
                    unsigned box_in, unsigned box_out, CUtensorMapSwizzle sw, CUtensorMap* out) {
  typedef CUresult (*Encode)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (Encode) nullptr;
    return (Encode)fn;
  }();
  if (!encode) return false;
  struct Entry {
    void* base;
    unsigned long long inner, outer;
    unsigned bi, bo;
    int sw;
    CUtensorMap map;
  };
  static thread_local Entry cache[16];
  static thread_local int next = 0;
  for (auto& e : cache)
    if (e.base == base && e.inner == inner && e.outer == outer && e.bi == box_in && e.bo == box_out && e.sw == (int)sw) {
      *out = e.map;
      return true;
    }
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * (unsigned long long)esize};
  cuuint32_t box[2] = {box_in, box_out};
  cuuint32_t es[2] = {1, 1};
  CUtensorMap m;
  if (encode(&m, dt, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  cache[next] = Entry{base, inner, outer, box_in, box_out, (int)sw, m};
  next = (next + 1) % 16;
  *out = m;
  return true;
}

__device__ __forceinline__ long long status_word(long long code, long long pos) { return (code << 60) | pos; }

__device__ __forceinline__ const uint8_t* page_ptr(const uint8_t* pool, const int32_t* table, int max_pages, int u,
                                                   int pg) {
  return pool + (size_t)table[(size_t)u * max_pages + pg] * PAGE;
}

}  // namespace akv
