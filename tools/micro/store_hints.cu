// Back-to-back streaming of the SoA shapes the mechanism kernels have, with
// different cache-policy hints on the loads and stores.  Question: can the
// steady-state rate of a read+write stream (each launch pays the write-back
// of the previous launch's dirty L2 lines) be raised by hints alone?
//   0 plain    : ld.global.nc          + st.global
//   1 st.cs    : ld.global.nc          + st.global.cs  (streaming store)
//   2 ld/st.cs : ld.global.cs          + st.global.cs
//   3 st.ef    : ld.global.nc          + st.global.L2::cache_hint (evict_first policy)
//   4 ld/st.ef : ld.global.nc.L2::cache_hint + st.global.L2::cache_hint (evict_first)
//   5 ld.lu    : ld.global.lu (last use) + st.global.cs
// R fp64 arrays read, W written per instance, one FMA-free sum per element.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o store_hints store_hints.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double ld(const double* p, int mode, unsigned long long pol) {
  double v;
  switch (mode) {
    case 2: v = __ldcs(p); break;
    case 4: asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol)); break;
    case 5: v = __ldlu(p); break;
    default: v = __ldg(p);
  }
  return v;
}
__device__ __forceinline__ void st(double* p, double v, int mode, unsigned long long pol) {
  switch (mode) {
    case 0: *p = v; break;
    case 3:
    case 4: asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory"); break;
    default: __stcs(p, v);
  }
}

template <int R, int W, int MODE>
__global__ void __launch_bounds__(256) soa(const double* __restrict__ in, double* __restrict__ out, long long n,
                                           long long pitch) {
  unsigned long long pol = 0;
  if (MODE == 3 || MODE == 4) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) s += ld(in + r * pitch + i, MODE, pol);
#pragma unroll
    for (int w = 0; w < W; ++w) st(out + w * pitch + i, s + w, MODE, pol);
  }
}

template <int R, int W, int MODE>
void run(long long n, double* in, double* out, long long pitch, int sms) {
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, soa<R, W, MODE>, 256, 0);
  long long want = (n + 255) / 256;
  int grid = (int)(want < (long long)per * sms ? want : (long long)per * sms);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int K = 40;
  for (int k = 0; k < 5; ++k) soa<R, W, MODE><<<grid, 256>>>(in, out, n, pitch);
  cudaEventRecord(a);
  for (int k = 0; k < K; ++k) soa<R, W, MODE><<<grid, 256>>>(in, out, n, pitch);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= K;
  const double bytes = 8.0 * (R + W) * n;
  printf("{\"mode\": %d, \"n\": %lld, \"R\": %d, \"W\": %d, \"us\": %.2f, \"GBps\": %.0f}\n", MODE, n, R, W, ms * 1e3,
         bytes / (ms * 1e-3) / 1e9);
}

template <int R, int W>
void all(long long n) {
  const long long pitch = (n + 31) / 32 * 32;
  double *in, *out;
  cudaMalloc(&in, R * pitch * 8);
  cudaMalloc(&out, W * pitch * 8);
  cudaMemset(in, 0, R * pitch * 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<R, W, 0>(n, in, out, pitch, sms);
  run<R, W, 1>(n, in, out, pitch, sms);
  run<R, W, 2>(n, in, out, pitch, sms);
  run<R, W, 3>(n, in, out, pitch, sms);
  run<R, W, 4>(n, in, out, pitch, sms);
  run<R, W, 5>(n, in, out, pitch, sms);
  cudaFree(in);
  cudaFree(out);
}

int main() {
  all<13, 6>(10000000);  // synapse-like: ~13 reads, ~6 writes
  all<10, 8>(10000000);  // hh shape
  all<6, 4>(3333333);    // BBP shape
  return 0;
}
