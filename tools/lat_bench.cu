// Dependent-latency microbenchmark for the instructions on the triangular
// solve's serial chain (one warp, clock64 around N dependent operations).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lat tools/lat_bench.cu && /tmp/lat
#include <cstdio>

constexpr int N = 4096;

__global__ void lat(double* out, long long* cyc, double seed) {
  __shared__ double sm[1024];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1.0 + 1e-9 * i;
  __syncwarp();
  double a = seed + lane, b = 1.0 - 1e-12 * lane;
  long long t0, t1;
  // (0) dependent DFMA
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) a = fma(a, b, 1e-300);
  t1 = clock64();
  cyc[0] = t1 - t0;
  // (1) dependent SHFL.IDX of a double (two 32-bit shuffles)
  double s = a;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) s = __shfl_sync(0xffffffffu, s, (lane + 1) & 31);
  t1 = clock64();
  cyc[1] = t1 - t0;
  // (2) dependent LDS (pointer chase through smem)
  int idx = lane;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) idx = static_cast<int>(sm[idx & 1023]) + (idx & 511);
  t1 = clock64();
  cyc[2] = t1 - t0;
  // (3) chain step as in trisolve: shfl from lane k, select, fma with smem
  double acc = a * 1e-3, zj = 0.0;
  t0 = clock64();
  for (int r = 0; r < N / 32; ++r) {
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const double zk = __shfl_sync(0xffffffffu, acc, k);
      if (lane == k) zj = zk;
      if (lane > k) acc = fma(-sm[k * 32 + lane], zk, acc);
    }
  }
  t1 = clock64();
  cyc[3] = t1 - t0;
  // (6) grouped chain: four pivots per step, 4x4 triangle redundantly
  double acc2 = a * 1e-3, zj2 = 0.0;
  const double* L = sm;
  t0 = clock64();
  for (int r = 0; r < N / 32; ++r) {
#pragma unroll
    for (int k = 0; k < 32; k += 4) {
      const double a0 = __shfl_sync(0xffffffffu, acc2, k);
      const double a1 = __shfl_sync(0xffffffffu, acc2, k + 1);
      const double a2 = __shfl_sync(0xffffffffu, acc2, k + 2);
      const double a3 = __shfl_sync(0xffffffffu, acc2, k + 3);
      const double z0 = a0;
      const double z1 = fma(-L[k * 33 + 1], z0, a1);
      const double z2 = fma(-L[k * 33 + 34], z1, fma(-L[k * 33 + 2], z0, a2));
      const double z3 = fma(-L[k * 33 + 67], z2, fma(-L[k * 33 + 35], z1, fma(-L[k * 33 + 3], z0, a3)));
      zj2 = lane == k ? z0 : (lane == k + 1 ? z1 : (lane == k + 2 ? z2 : (lane == k + 3 ? z3 : zj2)));
      if (lane > k + 3) {
        acc2 = fma(-L[k * 32 + lane], z0, acc2);
        acc2 = fma(-L[k * 32 + 32 + lane], z1, acc2);
        acc2 = fma(-L[k * 32 + 64 + lane], z2, acc2);
        acc2 = fma(-L[k * 32 + 96 + lane], z3, acc2);
      }
    }
  }
  t1 = clock64();
  cyc[6] = t1 - t0;
  // (4) DMUL chain
  double m = a;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) m = m * b;
  t1 = clock64();
  cyc[4] = t1 - t0;
  // (5) 32-bit SHFL chain
  int si = lane;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) si = __shfl_sync(0xffffffffu, si, (si + 1) & 31);
  t1 = clock64();
  cyc[5] = t1 - t0;
  out[threadIdx.x] = a + s + idx + acc + zj + m + si + acc2 + zj2;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 32 * sizeof(double));
  cudaMallocManaged(&cyc, 8 * sizeof(long long));
  for (int rep = 0; rep < 2; ++rep) {
    lat<<<1, 32>>>(out, cyc, 0.5);
    cudaDeviceSynchronize();
  }
  const char* names[] = {"DFMA", "SHFL.f64", "LDS chase", "chain step", "DMUL", "SHFL.b32", "chain4/row"};
  for (int i = 0; i < 7; ++i) printf("%-10s %.2f cycles/op\n", names[i], double(cyc[i]) / N);
  return 0;
}
