// rf_synth.cu -- measurement infrastructure: analytic-scene RGB-D renderer.
//
// Device counterpart of the reference's synthetic data generator
// (/root/reference/pkg/src/refusion/synth.py:46-283): unions of signed
// distance primitives (sphere, solid box, hollow room shell), sphere-traced
// z-depth with 256 steps / 1e-5 tolerance, flat-albedo Lambert colour and
// sigma0 * z^2 depth noise.  The CPU renderer takes 2.46 s per 640x480
// frame, which rules out the 2,000-20,000-frame configs; this
// kernel renders a frame in well under a millisecond.  It is NOT on the
// timed hot path and makes no bit-parity claim with synth.py (its noise
// stream is a counter-based hash, not numpy's PCG64).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "refusion_b200.h"

namespace {

constexpr int kSphere = 0, kRoom = 2;  // kind 1 = BoxSolid

__device__ __forceinline__ double prim_sdf(const rf_synth_prim& p, double x, double y, double z) {
  const double dx = x - p.center[0], dy = y - p.center[1], dz = z - p.center[2];
  if (p.kind == kSphere) return sqrt(dx * dx + dy * dy + dz * dz) - p.size[0];
  // box / room: synth.py:62-81
  const double qx = fabs(dx) - p.size[0], qy = fabs(dy) - p.size[1], qz = fabs(dz) - p.size[2];
  const double ox = fmax(qx, 0.0), oy = fmax(qy, 0.0), oz = fmax(qz, 0.0);
  const double outside = sqrt(ox * ox + oy * oy + oz * oz);
  const double inside = fmin(fmax(qx, fmax(qy, qz)), 0.0);
  const double s = outside + inside;
  return p.kind == kRoom ? -s : s;
}

__device__ __forceinline__ double scene_sdf(const rf_synth_prim* prims, int n, double x, double y,
                                            double z, int* which) {
  double best = 1e300;
  int arg = 0;
  for (int i = 0; i < n; ++i) {
    const double s = prim_sdf(prims[i], x, y, z);
    if (s < best) {
      best = s;
      arg = i;
    }
  }
  if (which) *which = arg;
  return best;
}

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double gauss(uint64_t seed, uint64_t idx) {
  const uint64_t a = mix(seed ^ mix(idx * 2 + 1));
  const uint64_t b = mix(seed ^ mix(idx * 2 + 2));
  const double u1 = (static_cast<double>(a >> 11) + 1.0) * (1.0 / 9007199254740993.0);
  const double u2 = static_cast<double>(b >> 11) * (1.0 / 9007199254740992.0);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

__global__ void k_render(const rf_synth_prim* __restrict__ prims_g, int n_prims, rf_pose pose,
                         double fx, double fy, double cx, double cy, int width, int height,
                         rf_synth_params sp, double* depth_out, double* color_out) {
  __shared__ rf_synth_prim prims[32];
  for (int i = threadIdx.x + threadIdx.y * blockDim.x; i < n_prims && i < 32;
       i += blockDim.x * blockDim.y)
    prims[i] = prims_g[i];
  __syncthreads();
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y * blockDim.y + threadIdx.y;
  if (u >= width || v >= height) return;
  const size_t pix = static_cast<size_t>(v) * width + u;
  // synth.py:220-250
  double dcx = (u - cx) / fx, dcy = (v - cy) / fy, dcz = 1.0;
  const double nrm = sqrt(dcx * dcx + dcy * dcy + dcz * dcz);
  dcx /= nrm;
  dcy /= nrm;
  dcz /= nrm;
  const double* R = pose.R;
  const double dwx = R[0] * dcx + R[1] * dcy + R[2] * dcz;
  const double dwy = R[3] * dcx + R[4] * dcy + R[5] * dcz;
  const double dwz = R[6] * dcx + R[7] * dcy + R[8] * dcz;
  const double t_cap = sp.z_max * nrm;
  double t = 0.0;
  bool hit = false;
  for (int s = 0; s < sp.steps; ++s) {
    const double d = scene_sdf(prims, n_prims, pose.t[0] + t * dwx, pose.t[1] + t * dwy,
                               pose.t[2] + t * dwz, nullptr);
    if (d < sp.tol) {
      hit = true;
      break;
    }
    t += fmax(d, 0.0);
    if (t > t_cap) break;
  }
  double depth = hit ? t * dcz : 0.0;
  if (depth > sp.z_max) depth = 0.0;
  const double clean = depth;
  if (depth > 0.0 && sp.sigma0 > 0.0) {  // synth.py:270-283
    depth = fmax(depth + gauss(sp.seed, pix) * sp.sigma0 * depth * depth, 0.0);
  }
  depth_out[pix] = depth;
  if (!color_out) return;
  double c0 = 0.0, c1 = 0.0, c2 = 0.0;
  if (clean > 0.0) {  // synth.py:253-267 (shaded at the noiseless hit point)
    const double px = pose.t[0] + t * dwx, py = pose.t[1] + t * dwy, pz = pose.t[2] + t * dwz;
    int which = 0;
    scene_sdf(prims, n_prims, px, py, pz, &which);
    const double e = 1e-4;
    double nx = scene_sdf(prims, n_prims, px + e, py, pz, nullptr) -
                scene_sdf(prims, n_prims, px - e, py, pz, nullptr);
    double ny = scene_sdf(prims, n_prims, px, py + e, pz, nullptr) -
                scene_sdf(prims, n_prims, px, py - e, pz, nullptr);
    double nz = scene_sdf(prims, n_prims, px, py, pz + e, nullptr) -
                scene_sdf(prims, n_prims, px, py, pz - e, nullptr);
    double nn = sqrt(nx * nx + ny * ny + nz * nz);
    if (nn == 0.0) nn = 1.0;
    nx /= nn;
    ny /= nn;
    nz /= nn;
    const double lam = sp.ambient + sp.diffuse * fmax(0.0, -(nx * sp.light[0] + ny * sp.light[1] +
                                                             nz * sp.light[2]));
    c0 = fmin(fmax(prims[which].albedo[0] * lam, 0.0), 255.0);
    c1 = fmin(fmax(prims[which].albedo[1] * lam, 0.0), 255.0);
    c2 = fmin(fmax(prims[which].albedo[2] * lam, 0.0), 255.0);
  }
  color_out[3 * pix] = c0;
  color_out[3 * pix + 1] = c1;
  color_out[3 * pix + 2] = c2;
}

}  // namespace

extern "C" rf_status rf_synth_render(const rf_synth_prim* prims_dev, int32_t n_prims,
                                     const rf_pose* pose, double fx, double fy, double cx,
                                     double cy, int32_t width, int32_t height,
                                     const rf_synth_params* params, double* depth_dev,
                                     double* color_dev, void* stream) {
  if (!prims_dev || n_prims <= 0 || n_prims > 32 || !pose || !params || !depth_dev ||
      width <= 0 || height <= 0)
    return RF_INVALID_ARG;
  dim3 block(16, 8);
  dim3 grid((width + 15) / 16, (height + 7) / 8);
  k_render<<<grid, block, 0, static_cast<cudaStream_t>(stream)>>>(
      prims_dev, n_prims, *pose, fx, fy, cx, cy, width, height, *params, depth_dev, color_dev);
  return cudaGetLastError() == cudaSuccess ? RF_OK : RF_CUDA;
}
