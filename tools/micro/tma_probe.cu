// Standalone check of the k_fuse keyframe-tile TMA path: a 2-D f64 tensor map
// over a 640x480 plane, 12x10 boxes loaded into shared memory by
// cp.async.bulk.tensor with an mbarrier, compared with direct reads.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <dlfcn.h>
#include <vector>

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__constant__ CUtensorMap c_tm;

template <int kVariant>
__global__ void k_probe(const __grid_constant__ CUtensorMap tm, const CUtensorMap* g_tm,
                        const double* plane, int W, int H, int* bad, int bw, int bh = 10) {
  __shared__ __align__(1024) double tile[16 * 16];
  __shared__ unsigned long long bar;
  const int neg = kVariant == 7 ? 0 : 3;
  const int x = blockIdx.x * 7 - neg, y = blockIdx.y * 5 - (neg ? 2 : 0);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (kVariant == 8) {  // warp-converged, predicated issue (the Triton form)
    const unsigned long long tma = reinterpret_cast<unsigned long long>(&tm);
    asm volatile(
        "{\n .reg .pred p;\n setp.eq.u32 p, %5, 0;\n"
        " @p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%4], %6;\n"
        " @p cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];\n}" ::"r"(smem_u32(tile)), "l"(tma), "r"(x), "r"(y),
        "r"(smem_u32(&bar)), "r"(threadIdx.x), "r"(bw * 8 * bh) : "memory");
  }
  if (threadIdx.x == 0 && kVariant != 8) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                 "r"(bw * 8 * bh) : "memory");
    unsigned long long tma = reinterpret_cast<unsigned long long>(&tm);
    if (kVariant == 2) tma = reinterpret_cast<unsigned long long>(g_tm);
    if (kVariant == 3) tma = reinterpret_cast<unsigned long long>(&c_tm);
    if (kVariant == 5) {
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                   " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(tile)), "l"(tma), "r"(x), "r"(y),
                   "r"(smem_u32(&bar)), "l"(0x1000000000000000ull) : "memory");
    } else if (kVariant == 6) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(tma) : "memory");
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                   " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(tile)), "l"(tma), "r"(x), "r"(y),
                   "r"(smem_u32(&bar)) : "memory");
    } else if (kVariant != 1)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                   " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(tile)), "l"(tma), "r"(x), "r"(y),
                   "r"(smem_u32(&bar)) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes"
                   " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(tile)), "l"(tma), "r"(x), "r"(y),
                   "r"(smem_u32(&bar)) : "memory");
  }
  unsigned ok = 0;
  while (!ok) {
    asm volatile("{\n .reg .pred P;\n mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n"
                 " selp.u32 %0, 1, 0, P;\n}" : "=r"(ok) : "r"(smem_u32(&bar)), "r"(0) : "memory");
  }
  for (int i = threadIdx.x; i < bh * bw; i += blockDim.x) {
    const int u = x + i % bw, v = y + i / bw;
    const double want = (u >= 0 && u < W && v >= 0 && v < H) ? plane[v * W + u] : 0.0;
    if (tile[i] != want) atomicAdd(bad, 1);
  }
}

int main() {
  const int W = 640, H = 480;
  std::vector<double> h(W * H);
  for (int i = 0; i < W * H; ++i) h[i] = 0.5 + i;
  double* d;
  int* bad;
  cudaMalloc(&d, sizeof(double) * W * H);
  cudaMalloc(&bad, sizeof(int));
  cudaMemcpy(d, h.data(), sizeof(double) * W * H, cudaMemcpyHostToDevice);
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);
  void* f = nullptr;
  if (std::getenv("DLSYM")) {
    void* h = dlopen("libcuda.so.1", RTLD_LAZY);
    f = dlsym(h, "cuTensorMapEncodeTiled");
  } else {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  }
  std::printf("encode fn %p\n", f);
  CUtensorMap m;
  const cuuint64_t dims[2] = {W, H};
  const cuuint64_t strides[1] = {W * 8};
  const int BW = std::getenv("BW") ? std::atoi(std::getenv("BW")) : 12;
  const int PROMO = std::getenv("PROMO") ? std::atoi(std::getenv("PROMO")) : 1;
  const int BH = std::getenv("BH") ? std::atoi(std::getenv("BH")) : 10;
  const int SWZ = std::getenv("SWZ") ? std::atoi(std::getenv("SWZ")) : 0;
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(BW), static_cast<cuuint32_t>(BH)};
  const cuuint32_t es[2] = {1, 1};
  const int DT = std::getenv("DT") ? std::atoi(std::getenv("DT")) : 0;
  const CUtensorMapDataType dt = DT == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT64
                                 : DT == 2 ? CU_TENSOR_MAP_DATA_TYPE_INT64
                                           : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  std::printf("sizeof(CUtensorMap) %zu align %zu\n", sizeof(CUtensorMap), alignof(CUtensorMap));
  CUresult r = reinterpret_cast<Encode>(f)(&m, dt, 2, d, dims, strides,
                                           box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                           static_cast<CUtensorMapSwizzle>(SWZ),
                                           PROMO ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                 : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  std::printf("encode %d\n", static_cast<int>(r));
  CUtensorMap* g_tm;
  cudaMalloc(&g_tm, sizeof(CUtensorMap));
  cudaMemcpy(g_tm, &m, sizeof(m), cudaMemcpyHostToDevice);
  cudaMemcpyToSymbol(c_tm, &m, sizeof(m));
  const int which = std::getenv("V") ? std::atoi(std::getenv("V")) : 0;
  for (int variant = which; variant <= which; ++variant) {
    cudaMemset(bad, 0, sizeof(int));
    if (variant == 0) k_probe<0><<<dim3(95, 98), 64>>>(m, g_tm, d, W, H, bad, BW, BH);
    else if (variant == 1) k_probe<1><<<dim3(95, 98), 64>>>(m, g_tm, d, W, H, bad, BW, BH);
    else if (variant == 2) k_probe<2><<<dim3(95, 98), 64>>>(m, g_tm, d, W, H, bad, BW, BH);
    else if (variant == 3) k_probe<3><<<dim3(95, 98), 64>>>(m, g_tm, d, W, H, bad, BW, BH);
    else if (variant == 5) k_probe<5><<<dim3(95, 98), 64>>>(m, g_tm, d, W, H, bad, BW, BH);
    else if (variant == 6) k_probe<6><<<dim3(95, 98), 64>>>(m, g_tm, d, W, H, bad, BW, BH);
    else if (variant == 7) k_probe<7><<<dim3(90, 94), 64>>>(m, g_tm, d, W, H, bad, BW, BH);
    else if (variant == 8) k_probe<8><<<dim3(95, 98), 64>>>(m, g_tm, d, W, H, bad, BW, BH);
    else {  // variant 4: variant 0 launched as 1-CTA clusters
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(95, 98);
      cfg.blockDim = dim3(64);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 1;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, k_probe<0>, m, (const CUtensorMap*)g_tm, (const double*)d, W, H, bad, BW, BH);
    }
    cudaError_t e = cudaDeviceSynchronize();
    int nb = -1;
    cudaMemcpy(&nb, bad, sizeof(int), cudaMemcpyDeviceToHost);
    std::printf("variant %d: %s, mismatches %d\n", variant, cudaGetErrorString(e), nb);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
