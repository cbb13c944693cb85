// Dependent-chain latency microbenchmarks on B200 (one warp), to size the
// simulation kernel's serial critical path.  nvcc -arch=sm_100a -O3 -fmad=false
#include <cstdio>
#include <cuda_runtime.h>

#define N 1024

__global__ void lat_dadd(double* out, long long* cyc, double a) {
  double x = a;
  const long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = __dadd_rn(x, a);
  const long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_dmul(double* out, long long* cyc, double a) {
  double x = a;
  const long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = __dmul_rn(x, a);
  const long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void thr_dadd4(double* out, long long* cyc, double a) {  // 4 independent chains
  double x = a, y = a * 2, z = a * 3, w = a * 4;
  const long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    x = __dadd_rn(x, a); y = __dadd_rn(y, a); z = __dadd_rn(z, a); w = __dadd_rn(w, a);
  }
  const long long t1 = clock64();
  out[threadIdx.x] = x + y + z + w;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_fadd(float* out, long long* cyc, float a) {
  float x = a;
  const long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = __fadd_rn(x, a);
  const long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_iadd64(long long* out, long long* cyc, long long a) {
  long long x = a;
  const long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = x * 3 + a;
  const long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_lds(double* out, long long* cyc, int s0) {
  __shared__ int idx[1024];
  for (int i = threadIdx.x; i < 1024; i += 32) idx[i] = (i * 7 + 1) & 1023;
  __syncwarp();
  int j = s0;
  const long long t0 = clock64();
  for (int i = 0; i < N; ++i) j = idx[j];
  const long long t1 = clock64();
  out[threadIdx.x] = j;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_redux(double* out, long long* cyc, unsigned a) {
  unsigned x = a + threadIdx.x;
  const long long t0 = clock64();
  for (int i = 0; i < N; ++i) x = __reduce_min_sync(0xffffffffu, x) + threadIdx.x;
  const long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_shfl(double* out, long long* cyc, double a) {
  double x = a + threadIdx.x;
  const long long t0 = clock64();
  for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
  const long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_ddiv(double* out, long long* cyc, double a) {
  double x = a;
  const long long t0 = clock64();
  for (int i = 0; i < N; ++i) x = __ddiv_rn(x, 1.0000001) + 0.5;
  const long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_dsetp_branch(double* out, long long* cyc, double a) {
  double x = a;
  int cnt = 0;
  const long long t0 = clock64();
  for (int i = 0; i < N; ++i) {
    x = __dadd_rn(x, a);
    if (x > 1e300) break;
    ++cnt;
  }
  const long long t1 = clock64();
  out[threadIdx.x] = x + cnt;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* od;
  long long* cy;
  cudaMalloc(&od, 1024 * 8);
  cudaMalloc(&cy, 8);
  long long h;
  auto run = [&](const char* name, auto launch, int ops) {
    for (int rep = 0; rep < 3; ++rep) launch();
    cudaDeviceSynchronize();
    cudaMemcpy(&h, cy, 8, cudaMemcpyDeviceToHost);
    printf("%-22s %8.2f cycles/op\n", name, double(h) / ops);
  };
  run("dadd latency", [&] { lat_dadd<<<1, 32>>>(od, cy, 1.0000001); }, N);
  run("dmul latency", [&] { lat_dmul<<<1, 32>>>(od, cy, 1.0000001); }, N);
  run("dadd 4 chains /step", [&] { thr_dadd4<<<1, 32>>>(od, cy, 1.0000001); }, N);
  run("fadd latency", [&] { lat_fadd<<<1, 32>>>((float*)od, cy, 1.0001f); }, N);
  run("imad64 latency", [&] { lat_iadd64<<<1, 32>>>((long long*)od, cy, 3); }, N);
  run("lds latency", [&] { lat_lds<<<1, 32>>>(od, cy, 1); }, N);
  run("redux+iadd latency", [&] { lat_redux<<<1, 32>>>(od, cy, 5); }, N);
  run("shfl latency", [&] { lat_shfl<<<1, 32>>>(od, cy, 1.0); }, N);
  run("ddiv+dadd latency", [&] { lat_ddiv<<<1, 32>>>(od, cy, 1.5); }, N);
  run("dadd+dsetp+bra /iter", [&] { lat_dsetp_branch<<<1, 32>>>(od, cy, 1.0000001); }, N);
  return 0;
}
