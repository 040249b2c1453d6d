// Streaming-read bandwidth of this GPU (the practical ceiling for a
// read-dominated kernel such as the triangular solve; MEASURED_PEAKS.json
// only has copy = read + write).  nvcc -O3 -gencode arch=compute_100a,code=sm_100a
//   tools/read_bw.cu -o tools/_read_bw && tools/_read_bw [GB]
#include <cstdio>
#include <cstdlib>

__global__ void read_kernel(const double2* __restrict__ p, size_t n, double* out) {
  double acc = 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const double2 v = __ldcs(p + i);
    acc += v.x + v.y;
  }
  if (acc == 1.2345) out[0] = acc;  // keep the loads
}

int main(int argc, char** argv) {
  const double gb = argc > 1 ? atof(argv[1]) : 16.0;
  const size_t bytes = (size_t)(gb * 1e9) & ~(size_t)31;
  double2* p;
  double* out;
  if (cudaMalloc(&p, bytes) != cudaSuccess) return 1;
  cudaMalloc(&out, 8);
  cudaMemset(p, 0, bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int per = 2; per <= 16; per *= 2) {
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      read_kernel<<<sms * per, 512>>>(p, bytes / 16, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("{\"ctas_per_sm\": %d, \"bytes\": %zu, \"ms\": %.4f, \"read_gbs\": %.1f}\n", per, bytes,
           best, bytes / (best * 1e-3) / 1e9);
  }
  return 0;
}
