#include <cstdio>
#include <cstdint>
__global__ void k(long long* out, double x0, double a, int reps, int64_t i0) {
  double x = x0; int64_t v = i0; unsigned u = threadIdx.x;
  long long t0 = clock64();
  // chain: DSETP -> branch
  int cnt = 0;
  for (int r = 0; r < reps; ++r) {
    if (x < a) { x = x * 1.0000001; cnt++; } else { x = x * 0.9999999; }
  }
  long long t1 = clock64();
  for (int r = 0; r < reps; ++r) {   // int64 compare -> branch
    if (v < 1000000000000ll) { v = v * 3 + 1; } else { v = v >> 1; }
  }
  long long t2 = clock64();
  for (int r = 0; r < reps; ++r) {   // ballot chain
    u = __ballot_sync(0xffffffffu, (u >> (threadIdx.x & 31)) & 1) + r;
  }
  long long t3 = clock64();
  for (int r = 0; r < reps; ++r) {   // redux chain
    u = __reduce_min_sync(0xffffffffu, u + threadIdx.x) + 1;
  }
  long long t4 = clock64();
  for (int r = 0; r < reps; ++r) {   // dadd chain
    x = __dadd_rn(x, 1e-9);
  }
  long long t5 = clock64();
  for (int r = 0; r < reps; ++r) {   // double bits -> int ops -> double
    int64_t b = __double_as_longlong(x);
    b = ((b >> 52) & 0x7ff) + (b & 0xfffffffffffffll) + 1;
    x = __longlong_as_double(b | 0x3ff0000000000000ll);
  }
  long long t6 = clock64();
  for (int r = 0; r < reps; ++r) {   // dsetp -> select (no branch)
    x = (x < a) ? x * 1.0000001 : x * 0.9999999;
  }
  long long t7 = clock64();
  for (int r = 0; r < reps; ++r) {   // 64-bit variable shift chain
    v = (v >> (r & 7)) + (v << 1) + r;
  }
  long long t8 = clock64();
  if (threadIdx.x == 0) {
    out[0] = (t1 - t0) / reps; out[1] = (t2 - t1) / reps; out[2] = (t3 - t2) / reps; out[3] = (t4 - t3) / reps;
    out[4] = (t5 - t4) / reps; out[5] = (t6 - t5) / reps; out[6] = (t7 - t6) / reps; out[7] = (t8 - t7) / reps;
    out[8] = cnt + (long long)x + v + u;
  }
}
int main() {
  long long* o; cudaMallocManaged(&o, 16 * sizeof(long long));
  k<<<1, 32>>>(o, 1.0, 1e300, 10000, 7);
  cudaDeviceSynchronize();
  const char* n[] = {"dsetp->branch", "isetp64->branch", "ballot chain", "redux chain", "dadd chain", "bits<->double int ops", "dsetp->select", "i64 shift chain"};
  for (int i = 0; i < 8; ++i) printf("%-24s %lld cycles/iter\n", n[i], o[i]);
}
