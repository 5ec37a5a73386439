// Streaming microbenchmark: how fast can one persistent CTA per SM pull HBM
// into the SM with each mechanism the kernels use?  (Measurement aid for the
// qk / pv ring design; not part of libakv.)
//
//   mode 0: TMA bulk ring   — 1 producer warp, NS stages of S bytes (one cp.async.bulk each),
//                             8 consumer warps wait full / arrive empty (+ touch 1 word)
//   mode 1: cp.async ring   — same ring, stage filled by 16-byte cp.async from 32 producer lanes
//   mode 2: direct loads    — 8 warps, ld.global.nc.v4 (16 B/lane), U loads in flight per lane
//   mode 3: TMA bulk ring, CHUNK-byte bulk copies (S/CHUNK per stage)
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench tools/ubench_stream.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
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
__device__ __forceinline__ void cpa16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa_arrive(uint64_t* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(b)) : "memory");
}

__global__ void __launch_bounds__(288, 1) ring_kernel(const uint8_t* src, size_t bytes, int S, int NS, int mode, int chunk,
                                                       unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)S * NS);
  uint64_t* empty = full + NS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], mode == 1 ? 33 : 1);
      mbar_init(&empty[i], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t nst = bytes / S;
  const size_t per = (nst + gridDim.x - 1) / gridDim.x;
  const size_t i0 = blockIdx.x * per, i1 = min(nst, i0 + per);
  if (warp == 0) {
    int k = 0;
    for (size_t i = i0; i < i1; ++i, ++k) {
      const int s = k % NS;
      wait(&empty[s], ((k / NS) & 1) ^ 1);
      const uint8_t* g = src + i * S;
      uint8_t* d = sm + (size_t)s * S;
      if (mode == 1) {
        for (int o = lane * 16; o < S; o += 512) cpa16(d + o, g + o);
        cpa_arrive(&full[s]);
        if (lane == 0) arrive(&full[s]);
      } else if (lane == 0) {
        expect_tx(&full[s], S);
        const int c = mode == 3 ? chunk : S;
        for (int o = 0; o < S; o += c) bulk(d + o, g + o, c, &full[s]);
      }
      __syncwarp();
    }
  } else {
    unsigned long long acc = 0;
    int k = 0;
    for (size_t i = i0; i < i1; ++i, ++k) {
      const int s = k % NS;
      wait(&full[s], (k / NS) & 1);
      acc += sm[(size_t)s * S + (warp * 32 + lane) * 4];
      __syncwarp();
      if (lane == 0) arrive(&empty[s]);
    }
    if (acc == 0x123456789ULL) sink[0] = acc;
  }
}

__global__ void __launch_bounds__(256) direct_kernel(const uint4* src, size_t n16, int U, unsigned long long* sink) {
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, nth = (size_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  size_t i = tid;
  for (; i + (size_t)(U - 1) * nth < n16; i += (size_t)U * nth) {
    uint4 v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u)
      if (u < U) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                              : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                              : "l"(src + i + u * nth));
#pragma unroll
    for (int u = 0; u < 16; ++u)
      if (u < U) acc ^= v[u].x ^ v[u].w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

int main() {
  const size_t bytes = 1ull << 30;
  uint8_t* buf[3];
  for (int i = 0; i < 3; ++i) {
    cudaMalloc(&buf[i], bytes);
    cudaMemset(buf[i], i + 1, bytes);
  }
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    for (int w = 0; w < 3; ++w) launch(buf[w % 3]);
    cudaEventRecord(e0);
    const int R = 9;
    for (int r = 0; r < R; ++r) launch(buf[r % 3]);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    printf("%-48s %8.1f GB/s  (%s)\n", name, bytes * (double)R / (ms * 1e-3) / 1e9, cudaGetErrorString(err));
  };
  char nm[128];
  struct Cfg { int mode, S, NS, chunk; };
  Cfg cfgs[] = {{0, 16384, 6, 0}, {0, 32768, 6, 0}, {0, 16384, 12, 0}, {0, 8192, 24, 0}, {0, 32768, 3, 0},
                {0, 65536, 3, 0}, {1, 16384, 6, 0}, {1, 32768, 6, 0}, {1, 16384, 12, 0}, {3, 32768, 6, 4096},
                {3, 32768, 6, 1024}, {3, 16384, 12, 2048}};
  for (const Cfg& c : cfgs) {
    snprintf(nm, sizeof nm, "ring mode %d S=%d NS=%d chunk=%d", c.mode, c.S, c.NS, c.chunk);
    const size_t smem = (size_t)c.S * c.NS + 16 * c.NS;
    run(nm, [&](uint8_t* b) { ring_kernel<<<sms, 288, smem>>>(b, bytes, c.S, c.NS, c.mode, c.chunk, sink); });
  }
  for (int U : {1, 2, 4, 8, 16}) {
    for (int bpsm : {1, 2, 4, 8}) {
      snprintf(nm, sizeof nm, "direct ld.v4 U=%d blocks/SM=%d", U, bpsm);
      run(nm, [&](uint8_t* b) { direct_kernel<<<sms * bpsm, 256>>>((const uint4*)b, bytes / 16, U, sink); });
    }
  }
  return 0;
}
