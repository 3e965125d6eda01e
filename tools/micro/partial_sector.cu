// Microbenchmark: DRAM traffic of 16-byte (half-sector) writes on B200 HBM3e.
// A: read every 16-B pair, write back the even pairs (half of each sector)
// B: read every pair, write back every pair
// C: no read, write the even pairs only
// D: read the even pairs only, write them back
// Run under ncu with dram__bytes_read.sum / dram__bytes_write.sum.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_rw(double2* buf, long long n, int mode) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const bool even = (i & 1) == 0;
    double2 v = make_double2(0.0, 0.0);
    if (mode == 0 || mode == 1 || (mode == 3 && even)) v = buf[i];
    v.x += 1.0;
    if (mode == 1 || even) buf[i] = v;
  }
}

int main() {
  const long long bytes = 1LL << 30, n = bytes / 16;
  double2* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 0, bytes);
  void* flush;
  cudaMalloc(&flush, 512 << 20);
  for (int mode = 0; mode < 4; ++mode) {
    cudaMemset(flush, mode, 512 << 20);  // evict L2
    k_rw<<<148 * 8, 256>>>(buf, n, mode);
    cudaDeviceSynchronize();
  }
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
