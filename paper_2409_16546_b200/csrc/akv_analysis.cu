// relative_error_histogram on device: the Table-1 buckets
// {0}, (0,1/1024), [1/1024,1/512), [1/512,1/256), [1/256,1/128), [1/128,inf)
// over n (test, ref) pairs.  Optional fp16 output grid first (SURVEY App. A
// A-hist, HB:187-190 float16_round: RNE to half).  ref = 0: test = 0 -> {0},
// else [1/128,inf).  The ratio is formed in fp64 like the oracle (identical
// IEEE division), so bucket counts are exact integers equal to the oracle's.
#include <algorithm>

#include "akv_common.cuh"

namespace akv {

__device__ __forceinline__ int err_bucket(double t, double r) {
  if (r == 0.0) return t == 0.0 ? 0 : 5;
  const double rel = fabs(t - r) / fabs(r);
  if (rel == 0.0) return 0;
  if (rel < 0x1p-10) return 1;
  if (rel < 0x1p-9) return 2;
  if (rel < 0x1p-8) return 3;
  if (rel < 0x1p-7) return 4;
  return 5;
}

__global__ void __launch_bounds__(256) error_hist_kernel(const float* __restrict__ test, const float* __restrict__ ref,
                                                         long long n, int fp16_round, unsigned long long* counts) {
  __shared__ unsigned int hist[6];
  if (threadIdx.x < 6) hist[threadIdx.x] = 0;
  __syncthreads();
  unsigned int local[6] = {0, 0, 0, 0, 0, 0};
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float t = test[i], r = ref[i];
    if (fp16_round) {
      t = __half2float(__float2half_rn(t));
      r = __half2float(__float2half_rn(r));
    }
    const int b = err_bucket((double)t, (double)r);
#pragma unroll
    for (int k = 0; k < 6; ++k) local[k] += (b == k);
  }
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const int s = warp_sum_i((int)local[k]);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(&hist[k], (unsigned)s);
  }
  __syncthreads();
  if (threadIdx.x < 6 && hist[threadIdx.x]) atomicAdd(counts + threadIdx.x, (unsigned long long)hist[threadIdx.x]);
}

}  // namespace akv

extern "C" int akv_error_histogram(const float* test, const float* ref, int64_t n, int32_t fp16_round,
                                   int64_t* counts, void* stream) {
  if (n < 0 || !counts || (n > 0 && (!test || !ref))) return AKV_EINVAL;
  cudaStream_t cs = (cudaStream_t)stream;
  if (cudaMemsetAsync(counts, 0, 6 * sizeof(int64_t), cs) != cudaSuccess) return AKV_ECUDA;
  if (n == 0) return AKV_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long blocks = std::min<long long>((n + 255) / 256, (long long)sms * 8);
  akv::error_hist_kernel<<<(int)blocks, 256, 0, cs>>>(test, ref, n, fp16_round,
                                                     reinterpret_cast<unsigned long long*>(counts));
  return cudaGetLastError() == cudaSuccess ? AKV_OK : AKV_ECUDA;
}
