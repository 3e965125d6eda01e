// Diagnostic: launch a Triton-compiled TMA kernel (tt_tma.cubin: 16x16 f64
// descriptor load at [16, 32] -> out) with a descriptor encoded here.
#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
int main() {
  cuInit(0);
  CUdevice dev; cuDeviceGet(&dev, 0);
  CUcontext ctx; cuDevicePrimaryCtxRetain(&ctx, dev); cuCtxSetCurrent(ctx);
  const char* path = std::getenv("CUBIN") ? std::getenv("CUBIN") : "tools/micro/tt_tma.cubin";
  FILE* f = std::fopen(path, "rb");
  std::vector<char> img(1 << 20);
  size_t n = std::fread(img.data(), 1, img.size(), f);
  std::fclose(f);
  img.resize(n);
  CUmodule mod; CUresult r = cuModuleLoadData(&mod, img.data());
  std::printf("load %d\n", r);
  const bool mine = std::getenv("CUBIN") != nullptr;
  const char* kname = std::getenv("KNAME") ? std::getenv("KNAME") : "kp0";
  CUfunction fn; r = cuModuleGetFunction(&fn, mod, mine ? kname : "k"); std::printf("getfn %s %d\n", kname, r);
  const int W = 640, H = 480;
  std::vector<double> h(W * H);
  for (int i = 0; i < W * H; ++i) h[i] = i;
  CUdeviceptr d, out;
  cuMemAlloc(&d, 8 * W * H); cuMemAlloc(&out, 8 * 256);
  cuMemcpyHtoD(d, h.data(), 8 * W * H);
  CUtensorMap m;
  const cuuint64_t dims[2] = {W, H};
  const cuuint64_t strides[1] = {W * 8};
  const cuuint32_t box[2] = {16, 16};
  const cuuint32_t es[2] = {1, 1};
  const int SWZ = std::getenv("SWZ") ? std::atoi(std::getenv("SWZ")) : 0;
  r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)d, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, (CUtensorMapSwizzle)SWZ,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  std::printf("encode %d\n", r);
  int s0 = H, s1 = W;
  long long t0 = W, t1 = 1;
  CUdeviceptr z = 0;
  void* args[] = {&m, &s0, &s1, &t0, &t1, &out, &z, &z};
  int Wv = W, Hv = H;
  CUdeviceptr badp; cuMemAlloc(&badp, 4); cuMemsetD32(badp, 0, 1);
  void* args2[] = {&m, &d, &Wv, &Hv, &badp};
  const int GX = std::getenv("GX") ? std::atoi(std::getenv("GX")) : 90;
  const int GY = std::getenv("GY") ? std::atoi(std::getenv("GY")) : 94;
  const int NT = std::getenv("NT") ? std::atoi(std::getenv("NT")) : 64;
  if (mine) r = cuLaunchKernel(fn, GX, GY, 1, NT, 1, 1, 4096, 0, args2, nullptr);
  else r = cuLaunchKernel(fn, 1, 1, 1, 128, 1, 1, 0, 0, args, nullptr);
  std::printf("launch %d\n", r);
  r = cuCtxSynchronize();
  const char* es_;
  cuGetErrorString(r, &es_);
  std::printf("sync %d %s\n", r, es_);
  std::vector<double> o(256);
  cuMemcpyDtoH(o.data(), out, 8 * 256);
  int bad = 0;
  if (mine) cuMemcpyDtoH(&bad, badp, 4);
  else for (int i = 0; i < 256; ++i) bad += o[i] != h[(16 + i / 16) * W + 32 + i % 16];
  std::printf("mismatches %d\n", bad);
  return 0;
}
