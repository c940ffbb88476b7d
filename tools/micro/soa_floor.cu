// Memory floor of the fused SoA step at the bench sizes: R fp64 arrays read,
// W written per instance, grid-stride, no arithmetic beyond a sum (so the
// loads cannot be elided).  Optionally F dependent FP64 FMAs per instance
// to see where the FP64 pipe starts to co-limit.  L2 flushed between launches.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o soa_floor soa_floor.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int R, int W, int F>
__global__ void __launch_bounds__(256) soa(const double* __restrict__ in, double* __restrict__ out, long long n, long long pitch) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double a[R];
#pragma unroll
    for (int r = 0; r < R; ++r) a[r] = __ldg(in + r * pitch + i);
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) s += a[r];
    // F/4 independent chains of 4-deep FMAs, ~like 3 gates of rate code
    double c0 = s, c1 = s * 0.5, c2 = s * 0.25, c3 = s * 0.125;
#pragma unroll
    for (int f = 0; f < F / 4; ++f) {
      c0 = fma(c0, 1.0000001, 1e-3); c1 = fma(c1, 0.9999999, 2e-3);
      c2 = fma(c2, 1.0000002, 3e-3); c3 = fma(c3, 0.9999998, 4e-3);
    }
    s = c0 + c1 + c2 + c3;
#pragma unroll
    for (int w = 0; w < W; ++w) out[w * pitch + i] = s + w;
  }
}

__global__ void flush(double* p, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) p[i] += 1.0;
}

template <int R, int W, int F>
void run(long long n, const char* tag) {
  const long long pitch = (n + 31) / 32 * 32;
  double *in, *out, *fl;
  cudaMalloc(&in, R * pitch * 8);
  cudaMalloc(&out, W * pitch * 8);
  const long long nf = 64ll << 20;  // 512 MB
  cudaMalloc(&fl, nf * 8);
  cudaMemset(in, 0, R * pitch * 8);
  int sms = 0, per = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, soa<R, W, F>, 256, 0);
  long long want = (n + 255) / 256;
  int grids[2] = {(int)(want < (long long)per * sms ? want : (long long)per * sms), (int)want};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int g = 0; g < 2; ++g) {
    float tot = 0;
    const int K = 30;
    for (int k = 0; k < K + 5; ++k) {
      flush<<<sms * 4, 256>>>(fl, nf);
      cudaEventRecord(a);
      soa<R, W, F><<<grids[g], 256>>>(in, out, n, pitch);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (k >= 5) tot += ms;
    }
    const double ms = tot / K;
    const double bytes = 8.0 * (R + W) * n;
    printf("{\"tag\": \"%s\", \"n\": %lld, \"R\": %d, \"W\": %d, \"F\": %d, \"grid\": \"%s\", \"us\": %.2f, \"GBps\": %.0f}\n", tag, n, R, W, F,
           g == 0 ? "persistent" : "one-per-thread", ms * 1e3, bytes / (ms * 1e-3) / 1e9);
  }
  cudaFree(in);
  cudaFree(out);
  cudaFree(fl);
}

int main() {
  run<10, 8, 0>(1000000, "hh-shape");
  run<10, 8, 64>(1000000, "hh-shape");
  run<10, 8, 192>(1000000, "hh-shape");
  run<10, 8, 352>(1000000, "hh-shape");
  run<6, 4, 0>(3333333, "NaTs2_t-shape");
  run<6, 4, 304>(3333333, "NaTs2_t-shape");
  run<6, 4, 0>(10000000, "big");
  return 0;
}
