// Dev microbenchmark: cycles per decode run of the simulation kernel's run
// block (4-way unrolled arrival-checked loop + single-step tail), one warp,
// runs chained through the clock.  nvcc -arch=sm_100a -O3 -fmad=false
#include <cstdio>

__device__ __forceinline__ int run4(double& clock, double& energy, double& flops, double& bytes,
                                    double d, double e, double f, double b, long ks, double a_h) {
  long j = 0;
  while (j + 4 <= ks) {
    const double c1 = __dadd_rn(clock, d);
    const double c2 = __dadd_rn(c1, d);
    const double c3 = __dadd_rn(c2, d);
    if (!(clock < a_h && c1 < a_h && c2 < a_h && c3 < a_h)) break;
    clock = __dadd_rn(c3, d);
    energy = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(energy, e), e), e), e);
    flops = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(flops, f), f), f), f);
    bytes = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(bytes, b), b), b), b);
    j += 4;
  }
  while (j < ks && clock < a_h) {
    clock = __dadd_rn(clock, d);
    energy = __dadd_rn(energy, e);
    flops = __dadd_rn(flops, f);
    bytes = __dadd_rn(bytes, b);
    ++j;
  }
  return int(j);
}

__device__ __forceinline__ int run_clock_only(double& clock, double d, long ks, double a_h) {
  long j = 0;
  while (j + 4 <= ks) {
    const double c3 = __dadd_rn(__dadd_rn(__dadd_rn(clock, d), d), d);
    if (!(c3 < a_h)) break;
    clock = __dadd_rn(c3, d);
    j += 4;
  }
  while (j < ks && clock < a_h) {
    clock = __dadd_rn(clock, d);
    ++j;
  }
  return int(j);
}

__global__ void bench(long long* cyc, double* sink, int reps, int k) {
  double clock = 1000.0 + threadIdx.x * 1e-12, energy = 5.0, flops = 1e12, bytes = 1e9;
  const double d = 0.0123456, e = 1.5, f = 3.0e9, b = 7.0e6;
  long total = 0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    const double a_h = clock + d * (k - 0.5);  // arrival inside the run: stops after k
    total += run4(clock, energy, flops, bytes, d, e, f, b, 1000, a_h);
  }
  long long t1 = clock64();
  for (int r = 0; r < reps; ++r) {
    const double a_h = clock + d * (k - 0.5);
    total += run_clock_only(clock, d, 1000, a_h);
  }
  long long t2 = clock64();
  sink[threadIdx.x] = clock + energy + flops + bytes + double(total);
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / reps;
    cyc[1] = (t2 - t1) / reps;
  }
}

int main() {
  long long* cyc;
  double* sink;
  cudaMallocManaged(&cyc, 2 * sizeof(long long));
  cudaMalloc(&sink, 32 * sizeof(double));
  for (int k : {3, 10, 20, 40}) {
    bench<<<1, 32>>>(cyc, sink, 2000, k);
    cudaDeviceSynchronize();
    std::printf("k=%2d  run4(clock+3 accumulators)=%lld cycles  clock-only=%lld cycles\n", k, cyc[0], cyc[1]);
  }
  return 0;
}
