// Diagnostic kernels for tma_cubin (driver-API launch of nvcc-built TMA
// kernels): variant bits: 1 = destination in dynamic shared memory,
// 2 = issue by elect.sync in a converged warp (Triton's form).
#include <cuda.h>
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
template <int V>
__device__ void body(const CUtensorMap& tm, const double* plane, int W, int H, int* bad) {
  extern __shared__ __align__(1024) double dyn[];
  __shared__ __align__(1024) double stat[16 * 16];
  __shared__ unsigned long long bar;
  double* tile = (V & 1) ? dyn : stat;
  const int x = blockIdx.x * 7, y = blockIdx.y * 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                 "r"(16 * 16 * 8) : "memory");
  __syncthreads();
  const unsigned long long tma = reinterpret_cast<unsigned long long>(&tm);
  if (V & 2) {
    if (threadIdx.x < 32)
      asm volatile(
          "{\n .reg .pred e;\n .reg .b32 r;\n elect.sync r|e, -1;\n"
          " @e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3}], [%4];\n}" ::"r"(smem_u32(tile)), "l"(tma), "r"(x), "r"(y),
          "r"(smem_u32(&bar)) : "memory");
  } else if (threadIdx.x == 0) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(tile)), "l"(tma), "r"(x), "r"(y),
                 "r"(smem_u32(&bar)) : "memory");
  }
  unsigned ok = 0;
  while (!ok) {
    asm volatile("{\n .reg .pred P;\n mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n"
                 " selp.u32 %0, 1, 0, P;\n}" : "=r"(ok) : "r"(smem_u32(&bar)), "r"(0) : "memory");
  }
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    const int u = x + i % 16, v = y + i / 16;
    const double want = (u < W && v < H) ? plane[v * W + u] : 0.0;
    if (tile[i] != want) atomicAdd(bad, 1);
  }
}
extern "C" __global__ void kp0(const __grid_constant__ CUtensorMap tm, const double* p, int W, int H, int* b) { body<0>(tm, p, W, H, b); }
extern "C" __global__ void kp1(const __grid_constant__ CUtensorMap tm, const double* p, int W, int H, int* b) { body<1>(tm, p, W, H, b); }
extern "C" __global__ void kp2(const __grid_constant__ CUtensorMap tm, const double* p, int W, int H, int* b) { body<2>(tm, p, W, H, b); }
extern "C" __global__ void kp3(const __grid_constant__ CUtensorMap tm, const double* p, int W, int H, int* b) { body<3>(tm, p, W, H, b); }
