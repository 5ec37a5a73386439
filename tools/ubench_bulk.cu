// Per-warp ring microbenchmark (measurement aid for the qk / pv redesign; not part of libakv):
// how fast do W warps per SM stream HBM into shared memory when every warp is its own
// producer (the pv3 pattern), as a function of the copy granularity?
//
//   mode 0: each stage = S/C bulk copies of C bytes (cp.async.bulk, UBLKCP), issued by lanes 0..S/C-1
//   mode 1: each stage = S/512 TMA gather4 copies (cp.async.bulk.tensor.2d tile::gather4, UTMALDG) of
//           4 rows x 128 B chosen from a 2-D [rows][128 B] view (rows picked with a stride, so the
//           four rows are not adjacent)
//   mode 2: direct ld.global.nc.v4 into registers, U 16-byte loads in flight per lane (no smem)
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_bulk tools/ubench_bulk.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t par) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
                   smem_u32(b)),
               "r"(par)
               : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
               "l"(src), "r"(n), "r"(smem_u32(b))
               : "memory");
}
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* tm, int x, int r0, int r1, int r2, int r3,
                                        uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(x), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(b))
      : "memory");
}

__global__ void ring(const uint8_t* src, size_t bytes, int S, int NS, int C, int mode, int U,
                     const __grid_constant__ CUtensorMap tm, unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
  uint8_t* ring = sm + (size_t)warp * (S * NS + 64);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + S * NS);
  const size_t gw = (size_t)blockIdx.x * nwarp + warp, nw = (size_t)gridDim.x * nwarp;
  const size_t nst = bytes / S, per = (nst + nw - 1) / nw;
  const size_t i0 = gw * per, i1 = min(nst, i0 + per);
  unsigned long long acc = 0;
  if (mode == 2) {
    // direct loads: each lane U x 16 B in flight, stage = 512*U bytes per warp step
    const size_t step = 512ull * U;
    const size_t b0 = i0 * S, b1 = i1 * S;
    for (size_t o = b0; o < b1; o += step) {
      uint4 v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u)
        if (u < U) {
          const uint8_t* p = src + o + (size_t)u * 512 + lane * 16;
          asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                       : "l"(p));
        }
#pragma unroll
      for (int u = 0; u < 16; ++u)
        if (u < U) acc += v[u].x ^ v[u].w;
    }
    if (acc == 0x1234567) sink[0] = acc;
    return;
  }
  if (lane == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const int rows_total = (int)(bytes / 128);
  auto issue = [&](size_t i, int slot) {
    uint8_t* dst = ring + (size_t)slot * S;
    if (lane == 0) expect_tx(&full[slot], S);
    __syncwarp();
    if (mode == 0) {
      const int n = S / C;
      for (int c = lane; c < n; c += 32) bulk(dst + c * C, src + i * S + (size_t)c * C, C, &full[slot]);
    } else {
      const int n = S / 512;  // gather4 instructions per stage
      for (int c = lane; c < n; c += 32) {
        // 4 rows spread over the stage's region of the buffer (stride 3 rows, wrapped)
        const int base = (int)((i * S) / 128) + 4 * c;
        const int r0 = base, r1 = base + 1, r2 = base + 2, r3 = base + 3;
        gather4(dst + c * 512, &tm, 0, r0 % rows_total, r1 % rows_total, r2 % rows_total, r3 % rows_total, &full[slot]);
      }
    }
  };
  int k = 0;
  size_t ii = i0;
  for (; k < NS - 1 && ii < i1; ++k, ++ii) issue(ii, k % NS);
  for (size_t i = i0; i < i1; ++i) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (ii < i1) {
      issue(ii, k % NS);
      ++ii;
      ++k;
    }
    const int slot = (int)((i - i0) % NS);
    mwait(&full[slot], (uint32_t)(((i - i0) / NS) & 1));
    acc += *reinterpret_cast<const uint32_t*>(ring + (size_t)slot * S + lane * 4);
    __syncwarp();
  }
  if (acc == 0x1234567) sink[0] = acc;
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const size_t bytes = 4ull << 30;
  uint8_t* src;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {128, bytes / 128};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {128, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = ((EncodeTiled)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, src, dims, strides, box, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("tensor map encode: %d\n", (int)r);
  cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  struct Cfg {
    int mode, S, NS, C, warps_per_cta, ctas_per_sm, U;
  };
  const Cfg cfgs[] = {
      {0, 8192, 2, 8192, 4, 3, 0},  {0, 8192, 2, 1024, 4, 3, 0}, {0, 8192, 2, 512, 4, 3, 0},
      {0, 8192, 2, 128, 4, 3, 0},   {0, 4096, 3, 4096, 4, 4, 0}, {0, 4096, 3, 512, 4, 4, 0},
      {0, 4096, 3, 128, 4, 4, 0},   {0, 2048, 4, 2048, 4, 6, 0}, {0, 2048, 4, 128, 4, 6, 0},
      {0, 16384, 3, 16384, 2, 2, 0}, {0, 4096, 4, 4096, 4, 3, 0}, {0, 4096, 3, 4096, 8, 2, 0},
      {1, 8192, 2, 512, 4, 3, 0},   {1, 4096, 3, 512, 4, 4, 0},  {1, 2048, 4, 512, 4, 6, 0},
      {2, 8192, 0, 0, 4, 3, 4},     {2, 8192, 0, 0, 4, 4, 8},    {2, 8192, 0, 0, 8, 2, 16},
  };
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (const Cfg& c : cfgs) {
    const int smem = c.mode == 2 ? 0 : c.warps_per_cta * (c.S * c.NS + 64);
    const int grid = sms * c.ctas_per_sm;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      ring<<<grid, 32 * c.warps_per_cta, smem>>>(src, bytes, c.S, c.NS, c.C, c.mode, c.U, tm, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ring, 32 * c.warps_per_cta, smem);
    printf("mode %d S %5d NS %d C %5d warps/cta %d ctas/sm %d (occ %d) U %2d: %7.1f GB/s %s\n", c.mode, c.S, c.NS, c.C,
           c.warps_per_cta, c.ctas_per_sm, occ, c.U, bytes / (ms * 1e-3) / 1e9, err ? cudaGetErrorString(err) : "");
  }
  return 0;
}
