// Measured FP64 pipe peak of this B200 (the FP64 roofline denominator; the
// driver-written MEASURED_PEAKS.json has HBM and bf16 only).
//
// Every thread runs CHAINS independent DFMA chains (enough ILP to hide the
// DFMA latency at full occupancy), grid = SMs x resident CTAs, timed with
// CUDA events after warm-up, best of REPS.  Reported as FP64 pipe
// instructions per second (one DFMA = one instruction = 2 flops) and per SM
// per clock, with the SM clock read from NVML-free cudaDevAttrClockRate and
// from %clock64 / %globaltimer inside the kernel (the clock it actually ran).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void __launch_bounds__(256) dfma_chains(double* out, int iters, double a, double b,
                                                   unsigned long long* clk) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3 + c;
  unsigned long long c0 = 0, t0 = 0;
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c0));
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 1234.5) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long c1, t1;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c1));
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    clk[0] = c1 - c0;
    clk[1] = t1 - t0;
  }
}

template <int CHAINS>
void run(int sms) {
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, dfma_chains<CHAINS>, 256, 0);
  const int grid = per * sms;
  double* out;
  unsigned long long* clk;
  cudaMalloc(&out, (size_t)grid * 256 * 8);
  cudaMallocManaged(&clk, 16);
  const int iters = 20000;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) dfma_chains<CHAINS><<<grid, 256>>>(out, iters, 0.999999, 1e-9, clk);
  cudaDeviceSynchronize();
  float best = 1e30f;
  double mhz = 0;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(a);
    dfma_chains<CHAINS><<<grid, 256>>>(out, iters, 0.999999, 1e-9, clk);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) {
      best = ms;
      mhz = (double)clk[0] / ((double)clk[1] * 1e-3);
    }
  }
  const double instr = (double)grid * 256 * iters * CHAINS;
  const double rate = instr / (best * 1e-3);
  printf("{\"chains\": %d, \"ctas_per_sm\": %d, \"grid\": %d, \"ms\": %.4f, \"dfma_per_s\": %.4e, "
         "\"tflops_fp64\": %.3f, \"sm_mhz_in_kernel\": %.0f, \"dfma_per_sm_per_clk\": %.2f}\n",
         CHAINS, per, grid, best, rate, 2 * rate / 1e12, mhz, rate / sms / (mhz * 1e6));
  cudaFree(out);
  cudaFree(clk);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<4>(sms);
  run<8>(sms);
  run<16>(sms);
  return 0;
}
