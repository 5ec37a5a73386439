// Layout probe for the qk9 tensor-core path (tcgen05 on sm_100a): D[128 x 16] (TMEM, fp32)
// = A[128 x K] (smem, fp16, MN-major, no swizzle, M-group stride SBO) x B[K x 16] (smem,
// fp16, K-major, no swizzle), K = 32 as two K = 16 MMAs, accumulator read back with
// tcgen05.ld.32x32b.x16.  Checks against a CPU product and prints the max error.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/ubench_umma tools/ubench_umma.cu && /tmp/ubench_umma
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>

constexpr int M = 128, N = 16, K = 32;
constexpr int SBO_A = (K / 8) * 128 + 16;  // M-group stride (bytes), padded off the bank period
constexpr int LBO_A = 128;                 // K-group stride
constexpr int SBO_B = 128;                 // N-group stride
constexpr int LBO_B = 256;                 // K-group stride (two N-groups of 128 B)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm_100)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

__global__ void probe(const __half* A, const __half* B, float* D, int a_major_mn) {
  __shared__ __align__(1024) uint8_t sa[(M / 8) * SBO_A];
  __shared__ __align__(1024) uint8_t sb[(K / 8) * LBO_B];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // A (m, k) at (m/8) SBO + (k/8) LBO + (k%8) 16 + (m%8) 2
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    *reinterpret_cast<__half*>(sa + (m / 8) * SBO_A + (k / 8) * LBO_A + (k % 8) * 16 + (m % 8) * 2) = A[m * K + k];
  }
  // B (n, k) at (k/8) LBO + (n/8) SBO + (n%8) 16 + (k%8) 2
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    *reinterpret_cast<__half*>(sb + (k / 8) * LBO_B + (n / 8) * SBO_B + (n % 8) * 16 + (k % 8) * 2) = B[n * K + k];
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tbase;
  if (tid == 0) {
    // kind::f16: D f32 (bits 4-5 = 1), A/B f16, a_major bit 15, N >> 3 at 17, M >> 4 at 24
    const uint32_t idesc = (1u << 4) | ((uint32_t)a_major_mn << 15) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    for (int kb = 0; kb < K / 16; ++kb) {
      const uint64_t da = desc(smem_u32(sa) + kb * 2 * LBO_A, LBO_A, SBO_A);
      const uint64_t db = desc(smem_u32(sb) + kb * 2 * LBO_B, LBO_B, SBO_B);
      const uint32_t acc = kb > 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
          "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
  }
  // wait for the commit
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
      "@!P1 bra WAIT;\n\t}" ::"r"(smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t r[16];
  const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  const int m = warp * 32 + lane;
  for (int n = 0; n < N; ++n) D[m * N + n] = __uint_as_float(r[n]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

int main() {
  __half *hA, *hB, *dA, *dB;
  float *hD, *dD;
  hA = (__half*)malloc(M * K * 2);
  hB = (__half*)malloc(N * K * 2);
  hD = (float*)malloc(M * N * 4);
  srand(1);
  for (int i = 0; i < M * K; ++i) hA[i] = __float2half((float)(rand() % 17 - 8) / 4.f);
  for (int i = 0; i < N * K; ++i) hB[i] = __float2half((float)(rand() % 13 - 6) / 8.f);
  cudaMalloc(&dA, M * K * 2);
  cudaMalloc(&dB, N * K * 2);
  cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, hA, M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, N * K * 2, cudaMemcpyHostToDevice);
  for (int mn = 1; mn >= 0; --mn) {
    cudaMemset(dD, 0, M * N * 4);
    probe<<<1, 128>>>(dA, dB, dD, mn);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("a_major_mn=%d: CUDA error %s\n", mn, cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(hD, dD, M * N * 4, cudaMemcpyDeviceToHost);
    double err = 0, mx = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += (double)__half2float(hA[m * K + k]) * (double)__half2float(hB[n * K + k]);
        err = fmax(err, fabs(ref - hD[m * N + n]));
        mx = fmax(mx, fabs(ref));
      }
    printf("a_major_mn=%d: max |err| = %g (max |ref| = %g) D[0][0..3] = %g %g %g %g\n", mn, err, mx, hD[0], hD[1],
           hD[2], hD[3]);
  }
  return 0;
}
