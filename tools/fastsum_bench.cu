// Dev microbenchmark: latency of psg_fastsum.cuh calls vs serial stepping
// (one warp, dependent chain, clock64).  nvcc -arch=sm_100a -O3 -fmad=false
#include <cstdio>
#include "../paper_2411_17651_b200/csrc/psg_fastsum.cuh"

__global__ void bench(double* out, long long* cyc, int reps, int k) {
  double acc = 1234.5678 + threadIdx.x * 1e-9, inc = 0.0123456789;
  double facc = 1.0e18 + 4096.0, finc = 3.0 * 1024 * 1024 * 7;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) acc = psg::fastsum::add_n(acc, inc, k);
  long long t1 = clock64();
  for (int r = 0; r < reps; ++r) facc = psg::fastsum::add_n(facc, finc, k);
  long long t2 = clock64();
  double c = acc;
  for (int r = 0; r < reps; ++r) psg::fastsum::advance_until(c, inc, k, c + inc * (k / 2) + 1e-7);
  long long t3 = clock64();
  double s = acc;
  for (int r = 0; r < reps; ++r)
    for (int j = 0; j < k; ++j) s = __dadd_rn(s, inc);
  long long t4 = clock64();
  out[threadIdx.x] = acc + facc + c + s;
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / reps;
    cyc[1] = (t2 - t1) / reps;
    cyc[2] = (t3 - t2) / reps;
    cyc[3] = (t4 - t3) / reps;
  }
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 32 * sizeof(double));
  cudaMallocManaged(&cyc, 4 * sizeof(long long));
  for (int k : {8, 32, 100, 1000}) {
    bench<<<1, 32>>>(out, cyc, 1000, k);
    cudaDeviceSynchronize();
    std::printf("k=%4d add_n(time-like)=%lld add_n(int-like)=%lld advance_until=%lld serial=%lld cycles\n",
                k, cyc[0], cyc[1], cyc[2], cyc[3]);
  }
  return 0;
}
