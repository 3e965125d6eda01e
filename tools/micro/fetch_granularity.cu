// Microbenchmark: DRAM bytes read when one 16-B pair is loaded per S bytes
// (S = 32, 64, 128), under the default L2 fetch granularity and with
// cudaLimitMaxL2FetchGranularity = 32 (argv[1] = 32 to set it).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void k_sparse_read(const double2* buf, long long n_pairs, int stride_pairs, double* out) {
  double acc = 0.0;
  for (long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * stride_pairs; i < n_pairs;
       i += (long long)gridDim.x * blockDim.x * stride_pairs)
    acc += buf[i].x;
  if (acc == 12345.0) *out = acc;
}

int main(int argc, char** argv) {
  if (argc > 1) {
    cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, atoi(argv[1]));
  }
  size_t g = 0;
  cudaDeviceGetLimit(&g, cudaLimitMaxL2FetchGranularity);
  printf("granularity %zu\n", g);
  const long long bytes = 1LL << 30, n = bytes / 16;
  double2* buf;
  double* out;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&out, 8);
  cudaMemset(buf, 0, bytes);
  void* flush;
  cudaMalloc(&flush, 512 << 20);
  for (int s : {2, 4, 8}) {  // one pair per 32, 64, 128 bytes
    cudaMemset(flush, s, 512 << 20);
    k_sparse_read<<<148 * 8, 256>>>(buf, n, s, out);
    cudaDeviceSynchronize();
  }
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
