// fp64 issue-rate microbenchmark for the interpreter's roofline (B200, sm_100a):
// DFMA, DADD and DMUL warp-instruction throughput with 8 independent chains
// per thread, all SMs busy.  Prints one JSON line: lane-operations per second
// (one DFMA = one lane-op = 2 flops) and the per-SM rate per clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu && ./fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 4096;

template <int OP>
__global__ void __launch_bounds__(256) k_fp64(double* out, double s) {
  double v[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) v[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      if (OP == 0) v[c] = fma(v[c], s, 0.5);
      else if (OP == 1) v[c] = v[c] + s;
      else v[c] = v[c] * s;
    }
  }
  double t = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) t += v[c];
  if (t == 123.456) out[0] = t;   // keep the work
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 8);
  const int blocks = sms * 8, threads = 256;
  const char* names[3] = {"dfma", "dadd", "dmul"};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  printf("{\"sms\": %d, \"max_clock_mhz\": %.0f", sms, clk / 1e3);
  for (int op = 0; op < 3; ++op) {
    auto run = [&] {
      if (op == 0) k_fp64<0><<<blocks, threads>>>(out, 0.999999);
      else if (op == 1) k_fp64<1><<<blocks, threads>>>(out, 1e-9);
      else k_fp64<2><<<blocks, threads>>>(out, 0.999999);
    };
    run();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) {
      cudaEventRecord(a);
      run();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    const double lane_ops = (double)blocks * threads * kIters * kChains;
    const double rate = lane_ops / (best * 1e-3);
    printf(", \"%s_lane_ops_per_s\": %.4e, \"%s_ms\": %.4f", names[op], rate, names[op], best);
  }
  printf("}\n");
  return 0;
}
