// rf_fusion.cu -- keyframe fusion on the device.
//
// Reference: /root/reference/pkg/src/refusion/keyframe_fusion.py
//   :142-231  normal_map / depth_sample_weight / discontinuity_mask  -> k_depth_weight
//   :238-276  fuse_depth: warp into the keyframe, np.add.at scatter, Eq. 1
//             -> k_warp, k_count, scan, k_scatter, k_merge (ordered segmented sums)
//   :278-346  grayscale / unsharp_mask / blurriness                  -> k_gauss_*, k_blur_*
//   :349-460  fuse_color: blur-weighted per-channel weighted median  -> k_fuse_color
//
// Arithmetic follows numpy / scipy operation by operation (compiled with
// -fmad=false): elementwise ufuncs are single IEEE ops, np.add.at applies
// in source order, scipy's correlate1d uses its symmetric-kernel loop,
// uniform_filter1d a running sum divided per output, and ndarray.sum()
// numpy's pairwise summation.  The one host-dependent step is
// geometry.transform (p @ R.T + t through BLAS): its multiply-add order is
// a parameter (rf_blas_order), calibrated on the host at start-up
// (keyframe_fusion.detect_blas_order).
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "refusion_b200.h"

namespace {


struct Intr {
  int w, h;
  double fx, fy, cx, cy;
};

// p @ R.T + t for one point, in the host BLAS's order (rf_blas_order)
__device__ __forceinline__ double blas_row(const double* r, double p0, double p1, double p2,
                                           int order) {
  switch (order) {
    case RF_BLAS_FMA_210: return fma(p2, r[2], fma(p1, r[1], p0 * r[0]));
    case RF_BLAS_FMA_012: return fma(p0, r[0], fma(p1, r[1], p2 * r[2]));
    case RF_BLAS_FMA_201: return fma(p2, r[2], fma(p0, r[0], p1 * r[1]));
    default: return (p0 * r[0] + p1 * r[1]) + p2 * r[2];
  }
}

__device__ __forceinline__ void transform(const rf_pose& T, double p0, double p1, double p2,
                                          int order, double& q0, double& q1, double& q2) {
  q0 = blas_row(T.R + 0, p0, p1, p2, order) + T.t[0];
  q1 = blas_row(T.R + 3, p0, p1, p2, order) + T.t[1];
  q2 = blas_row(T.R + 6, p0, p1, p2, order) + T.t[2];
}

// ---------------------------------------------------------------------------
// depth sample weight w_z = cos(theta) / Z^2 with the discontinuity mask

// normal_map (:142-188) at one pixel: central differences of unprojected
// neighbours; borders and pixels with an invalid neighbour get 0.
__device__ __forceinline__ void normal_at(const double* __restrict__ depth, const Intr& in, int u,
                                          int v, double& n0, double& n1, double& n2) {
  const int W = in.w, H = in.h;
  auto D = [&](int vv, int uu) { return __ldg(&depth[static_cast<size_t>(vv) * W + uu]); };
  auto dx = [&](int uu) { return (static_cast<double>(uu) - in.cx) / in.fx; };  // ray_grid
  auto dy = [&](int vv) { return (static_cast<double>(vv) - in.cy) / in.fy; };
  n0 = n1 = n2 = 0.0;
  if (u >= 1 && u <= W - 2 && v >= 1 && v <= H - 2) {
    const double d = D(v, u);
    const double dr = D(v, u + 1), dl = D(v, u - 1), dd = D(v + 1, u), du = D(v - 1, u);
    const double xr = dx(u + 1), xl = dx(u - 1), xc = dx(u);
    const double yc = dy(v), yd = dy(v + 1), yu = dy(v - 1);
    const double a0 = xr * dr - xl * dl, a1 = yc * dr - yc * dl, a2 = dr - dl;
    const double b0 = xc * dd - xc * du, b1 = yd * dd - yu * du, b2 = dd - du;
    const double c0 = a1 * b2 - a2 * b1;  // np.cross
    const double c1 = a2 * b0 - a0 * b2;
    const double c2 = a0 * b1 - a1 * b0;
    const double nrm = sqrt(c0 * c0 + c1 * c1 + c2 * c2);
    const bool ok = d > 0 && dr > 0 && dl > 0 && dd > 0 && du > 0 && nrm > 0;
    if (ok) {
      n0 = c0 / nrm;
      n1 = c1 / nrm;
      n2 = c2 / nrm;
    }
  }
}

__global__ void k_normal_map(const double* __restrict__ depth, Intr in, double* __restrict__ out) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y * blockDim.y + threadIdx.y;
  if (u >= in.w || v >= in.h) return;
  double n0, n1, n2;
  normal_at(depth, in, u, v, n0, n1, n2);
  double* o = out + 3 * (static_cast<size_t>(v) * in.w + u);
  o[0] = n0;
  o[1] = n1;
  o[2] = n2;
}

// depth_sample_weight with caller-supplied normals (:191-208)
__global__ void k_weight_from_normals(const double* __restrict__ depth,
                                      const double* __restrict__ normals, Intr in,
                                      double* __restrict__ w_out) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y * blockDim.y + threadIdx.y;
  if (u >= in.w || v >= in.h) return;
  const size_t i = static_cast<size_t>(v) * in.w + u;
  const double rx = (static_cast<double>(u) - in.cx) / in.fx;
  const double ry = (static_cast<double>(v) - in.cy) / in.fy;
  const double ray_norm = sqrt(rx * rx + ry * ry + 1.0);
  const double cos_t = (normals[3 * i] * rx + normals[3 * i + 1] * ry + normals[3 * i + 2]) / ray_norm;
  const double d = depth[i];
  w_out[i] = (d > 0 && isfinite(d) && cos_t > 0) ? cos_t / (d * d) : 0.0;
}

// flags: RF_DW_MASK applies the discontinuity mask to w (fuse_depth's
// w_map); RF_DW_MASK_ONLY writes the mask itself as 1.0 / 0.0.
__global__ void k_depth_weight(const double* __restrict__ depth, Intr in, double delta_disc,
                               int flags, double* __restrict__ w_out) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y * blockDim.y + threadIdx.y;
  if (u >= in.w || v >= in.h) return;
  const int W = in.w, H = in.h;
  auto D = [&](int vv, int uu) { return __ldg(&depth[static_cast<size_t>(vv) * W + uu]); };
  auto dx = [&](int uu) { return (static_cast<double>(uu) - in.cx) / in.fx; };  // ray_grid
  auto dy = [&](int vv) { return (static_cast<double>(vv) - in.cy) / in.fy; };
  const double d = D(v, u);
  double n0, n1, n2;
  normal_at(depth, in, u, v, n0, n1, n2);
  // depth_sample_weight (:191-208)
  const double rx = dx(u), ry = dy(v);
  const double ray_norm = sqrt(rx * rx + ry * ry + 1.0);
  const double cos_t = (n0 * rx + n1 * ry + n2) / ray_norm;
  double w = 0.0;
  if (d > 0 && isfinite(d) && cos_t > 0) w = cos_t / (d * d);
  // discontinuity_mask (:211-231): invalid, or next to invalid / a jump
  bool masked = !(d > 0);
  if (!masked) {
    for (int sv = -1; sv <= 1 && !masked; ++sv)
      for (int su = -1; su <= 1; ++su) {
        if (sv == 0 && su == 0) continue;
        const int nv = v + sv, nu = u + su;
        if (nv < 0 || nv >= H || nu < 0 || nu >= W) continue;
        const double nb = D(nv, nu);
        if (!(nb > 0) || fabs(d - nb) > delta_disc) {
          masked = true;
          break;
        }
      }
  }
  double out = w;
  if (flags & RF_DW_MASK_ONLY) out = masked ? 1.0 : 0.0;
  else if ((flags & RF_DW_MASK) && masked) out = 0.0;
  w_out[static_cast<size_t>(v) * W + u] = out;
}

// ---------------------------------------------------------------------------
// fuse_depth: warp -> ordered scatter -> Eq. 1

__global__ void k_warp(const double* __restrict__ depth, const double* __restrict__ w_map, Intr in,
                       rf_pose rel, int order, int* __restrict__ target,
                       double* __restrict__ val_wz, double* __restrict__ val_w,
                       int* __restrict__ counts) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = in.w * in.h;
  if (i >= n) return;
  int t = -1;
  const double ws = __ldg(&w_map[i]);
  if (ws > 0.0) {
    const int u = i % in.w, v = i / in.w;
    const double z = __ldg(&depth[i]);
    const double p0 = ((static_cast<double>(u) - in.cx) / in.fx) * z;
    const double p1 = ((static_cast<double>(v) - in.cy) / in.fy) * z;
    double q0, q1, q2;
    transform(rel, p0, p1, z, order, q0, q1, q2);
    if (q2 > 0) {
      const double uf = floor(in.fx * q0 / q2 + in.cx + 0.5);
      const double vf = floor(in.fy * q1 / q2 + in.cy + 0.5);
      if (uf >= 0 && uf < in.w && vf >= 0 && vf < in.h) {
        t = static_cast<int>(vf) * in.w + static_cast<int>(uf);
        val_wz[i] = ws * q2;
        val_w[i] = ws;
        atomicAdd(&counts[t], 1);
      }
    }
  }
  target[i] = t;
}

// fuse_depth's per-pixel front half in one pass (:245-269): the member's
// weight map w = depth_sample_weight masked by discontinuity_mask (the
// k_depth_weight arithmetic), the member's depth copy, then the warp of a
// weighted pixel into the keyframe (k_warp) -- target pixel, its two
// summands and the per-target count.
__global__ void k_dw_warp(const double* __restrict__ depth, Intr in, double delta_disc,
                          rf_pose rel, int order, double* __restrict__ w_map,
                          double* __restrict__ depth_copy, int* __restrict__ target,
                          double* __restrict__ val_wz, double* __restrict__ val_w,
                          int* __restrict__ counts) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y * blockDim.y + threadIdx.y;
  if (u >= in.w || v >= in.h) return;
  const int W = in.w, H = in.h;
  const size_t i = static_cast<size_t>(v) * W + u;
  auto D = [&](int vv, int uu) { return __ldg(&depth[static_cast<size_t>(vv) * W + uu]); };
  const double d = D(v, u);
  double n0, n1, n2;
  normal_at(depth, in, u, v, n0, n1, n2);
  const double rx = (static_cast<double>(u) - in.cx) / in.fx;
  const double ry = (static_cast<double>(v) - in.cy) / in.fy;
  const double ray_norm = sqrt(rx * rx + ry * ry + 1.0);
  const double cos_t = (n0 * rx + n1 * ry + n2) / ray_norm;
  double w = 0.0;
  if (d > 0 && isfinite(d) && cos_t > 0) w = cos_t / (d * d);
  bool masked = !(d > 0);
  if (!masked) {
    for (int sv = -1; sv <= 1 && !masked; ++sv)
      for (int su = -1; su <= 1; ++su) {
        if (sv == 0 && su == 0) continue;
        const int nv = v + sv, nu = u + su;
        if (nv < 0 || nv >= H || nu < 0 || nu >= W) continue;
        const double nb = D(nv, nu);
        if (!(nb > 0) || fabs(d - nb) > delta_disc) {
          masked = true;
          break;
        }
      }
  }
  if (masked) w = 0.0;
  w_map[i] = w;
  depth_copy[i] = d;
  int t = -1;
  if (w > 0.0) {  // k_warp
    const double p0 = ((static_cast<double>(u) - in.cx) / in.fx) * d;
    const double p1 = ((static_cast<double>(v) - in.cy) / in.fy) * d;
    double q0, q1, q2;
    transform(rel, p0, p1, d, order, q0, q1, q2);
    if (q2 > 0) {
      const double uf = floor(in.fx * q0 / q2 + in.cx + 0.5);
      const double vf = floor(in.fy * q1 / q2 + in.cy + 0.5);
      if (uf >= 0 && uf < in.w && vf >= 0 && vf < in.h) {
        t = static_cast<int>(vf) * in.w + static_cast<int>(uf);
        val_wz[i] = w * q2;
        val_w[i] = w;
        atomicAdd(&counts[t], 1);
      }
    }
  }
  target[i] = t;
}

__global__ void k_scatter(const int* __restrict__ target, int n, const int* __restrict__ offsets,
                          int* __restrict__ cursor, int* __restrict__ slots) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int t = target[i];
  if (t < 0) return;
  slots[offsets[t] + atomicAdd(&cursor[t], 1)] = i;
}

// np.add.at applies contributions in source order: sort each (short)
// segment by source index, sum sequentially, then the Eq. 1 merge
// (:270-276).
__global__ void k_merge(double* __restrict__ kf_depth, double* __restrict__ kf_weight, int n,
                        const int* __restrict__ counts, const int* __restrict__ offsets,
                        int* __restrict__ slots, const double* __restrict__ val_wz,
                        const double* __restrict__ val_w) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int c = counts[t];
  if (c == 0) return;
  int* seg = slots + offsets[t];
  for (int a = 1; a < c; ++a) {  // insertion sort by source index
    const int key = seg[a];
    int b = a - 1;
    while (b >= 0 && seg[b] > key) {
      seg[b + 1] = seg[b];
      --b;
    }
    seg[b + 1] = key;
  }
  double awz = 0.0, aw = 0.0;
  for (int a = 0; a < c; ++a) {
    awz = awz + val_wz[seg[a]];
    aw = aw + val_w[seg[a]];
  }
  if (aw > 0) {
    const double kd = kf_depth[t], kw = kf_weight[t];
    kf_depth[t] = (kd * kw + awz) / (kw + aw);
    kf_weight[t] = kw + aw;
  }
}

// ---------------------------------------------------------------------------
// colour prep: grayscale, unsharp mask (scipy gaussian_filter, mode
// 'nearest', separable: axis 0 then axis 1), blurriness

// scipy correlate1d, symmetric weights: out = x0*w0 + sum_{j=r..1} (x[-j] + x[+j]) * w[j]
__device__ __forceinline__ double corr_sym(const double* line, int stride, int len, int i,
                                           const double* w, int r) {
  double acc = line[static_cast<size_t>(i) * stride] * w[0];
  for (int j = r; j >= 1; --j) {
    const int lo = max(i - j, 0), hi = min(i + j, len - 1);  // mode 'nearest'
    acc = acc + (line[static_cast<size_t>(lo) * stride] + line[static_cast<size_t>(hi) * stride]) * w[j];
  }
  return acc;
}

struct GaussW {
  double w[16];  // w[0] centre, w[j] = weight at offset j
  int r;
};

// pass along axis 0 (vertical) on channel ch of an interleaved (h, w, c) image
__global__ void k_gauss_rows(const double* __restrict__ img, int W, int H, int C, GaussW g,
                             double* __restrict__ out) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y * blockDim.y + threadIdx.y;
  if (u >= W || v >= H) return;
  for (int ch = 0; ch < C; ++ch)
    out[(static_cast<size_t>(v) * W + u) * C + ch] =
        corr_sym(img + static_cast<size_t>(u) * C + ch, W * C, H, v, g.w, g.r);
}

// grayscale (:303-307) fused into the first (vertical) Gaussian pass, which
// reads the same frame colour
__global__ void k_gauss_rows_gray(const double* __restrict__ img, int W, int H, GaussW g,
                                  double* __restrict__ out, double* __restrict__ gray) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y * blockDim.y + threadIdx.y;
  if (u >= W || v >= H) return;
  const size_t px = static_cast<size_t>(v) * W + u;
  for (int ch = 0; ch < 3; ++ch)
    out[px * 3 + ch] = corr_sym(img + static_cast<size_t>(u) * 3 + ch, W * 3, H, v, g.w, g.r);
  const double* c = img + 3 * px;
  gray[px] = 0.299 * c[0] + 0.587 * c[1] + 0.114 * c[2];
}

// pass along axis 1, then unsharp: clip(img + gain * (img - low), 0, 255)
__global__ void k_gauss_cols_unsharp(const double* __restrict__ img,
                                     const double* __restrict__ tmp, int W, int H, int C,
                                     GaussW g, double gain, double* __restrict__ out) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y * blockDim.y + threadIdx.y;
  if (u >= W || v >= H) return;
  for (int ch = 0; ch < C; ++ch) {
    const size_t at = (static_cast<size_t>(v) * W + u) * C + ch;
    const double low = corr_sym(tmp + static_cast<size_t>(v) * W * C + ch, C, W, u, g.w, g.r);
    const double x = img[at];
    const double s = x + gain * (x - low);
    out[at] = fmin(fmax(s, 0.0), 255.0);  // np.clip (NaN-free inputs)
  }
}

__global__ void k_gray(const double* __restrict__ color, int n, double* __restrict__ gray) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* c = color + 3 * static_cast<size_t>(i);
  gray[i] = 0.299 * c[0] + 0.587 * c[1] + 0.114 * c[2];  // :307
}

// uniform_filter1d(size 9, mode 'nearest') along one axis: running sum,
// divided per output; then |diff(f)|, |diff(b)| and v = max(0, d_f - d_b)
// written flattened row-major for the pairwise sums.  One thread per line.
__global__ void k_blur_lines(const double* __restrict__ f, int W, int H, int axis, int size,
                             double* __restrict__ b, double* __restrict__ d_f,
                             double* __restrict__ vv) {
  const int line = blockIdx.x * blockDim.x + threadIdx.x;
  const int lines = axis == 0 ? W : H;
  if (line >= lines) return;
  const int len = axis == 0 ? H : W;
  const size_t stride = axis == 0 ? W : 1;
  const double* src = f + (axis == 0 ? line : static_cast<size_t>(line) * W);
  double* dst = b + (axis == 0 ? line : static_cast<size_t>(line) * W);
  const int s1 = size / 2;
  auto at = [&](int k) { return src[static_cast<size_t>(min(max(k, 0), len - 1)) * stride]; };
  double tmp = 0.0;
  for (int l = 0; l < size; ++l) tmp = tmp + at(l - s1);
  dst[0] = tmp / size;
  for (int l = 1; l < len; ++l) {
    tmp = tmp + (at(l + size - 1 - s1) - at(l - 1 - s1));
    dst[static_cast<size_t>(l) * stride] = tmp / size;
  }
  // diffs along the axis, flattened as numpy lays them out: (H-1, W) or (H, W-1)
  for (int l = 0; l + 1 < len; ++l) {
    const double df = fabs(src[static_cast<size_t>(l + 1) * stride] - src[static_cast<size_t>(l) * stride]);
    const double db = fabs(dst[static_cast<size_t>(l + 1) * stride] - dst[static_cast<size_t>(l) * stride]);
    const size_t o = axis == 0 ? static_cast<size_t>(l) * W + line : static_cast<size_t>(line) * (W - 1) + l;
    d_f[o] = df;
    vv[o] = fmax(0.0, df - db);
  }
}

// The same per line, one warp per line through shared memory: the lanes load
// the line (coalesced along rows), lane 0 runs the sequential running sum out
// of shared memory (scipy's order, so the bits match k_blur_lines), and the
// lanes then write the filtered line and its diffs in parallel.
constexpr int kBlurWarps = 4;
constexpr int kBlurMaxLen = 3072;  // 2 x 8 B x len per warp in dynamic smem

__global__ void __launch_bounds__(32 * kBlurWarps)
    k_blur_lines_smem(const double* __restrict__ f, int W, int H, int axis, int size,
                      double* __restrict__ b, double* __restrict__ d_f,
                      double* __restrict__ vv) {
  extern __shared__ double s_blur[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int line = blockIdx.x * kBlurWarps + warp;
  const int lines = axis == 0 ? W : H;
  if (line >= lines) return;
  const int len = axis == 0 ? H : W;
  const size_t stride = axis == 0 ? W : 1;
  const double* src = f + (axis == 0 ? line : static_cast<size_t>(line) * W);
  double* dst = b + (axis == 0 ? line : static_cast<size_t>(line) * W);
  double* s_in = s_blur + static_cast<size_t>(warp) * 2 * len;
  double* s_out = s_in + len;
  for (int k = lane; k < len; k += 32) s_in[k] = src[static_cast<size_t>(k) * stride];
  __syncwarp();
  const int s1 = size / 2;
  auto at = [&](int k) { return s_in[min(max(k, 0), len - 1)]; };
  // the running sum's increments (x[l+size-1-s1] - x[l-1-s1]), rounded as
  // scipy rounds them, computed by all lanes; lane 0 then only chains adds
  for (int l = 1 + lane; l < len; l += 32) s_out[l] = at(l + size - 1 - s1) - at(l - 1 - s1);
  __syncwarp();
  if (lane == 0) {  // the running sums (sequential); the lanes divide below
    double tmp = 0.0;
    for (int l = 0; l < size; ++l) tmp = tmp + at(l - s1);
    s_out[0] = tmp;
#pragma unroll 16
    for (int l = 1; l < len; ++l) {
      tmp = tmp + s_out[l];
      s_out[l] = tmp;
    }
  }
  __syncwarp();
  for (int l = lane; l < len; l += 32) s_out[l] = s_out[l] / size;
  __syncwarp();
  for (int l = lane; l < len; l += 32) {
    dst[static_cast<size_t>(l) * stride] = s_out[l];
    if (l + 1 < len) {
      const double df = fabs(s_in[l + 1] - s_in[l]);
      const double db = fabs(s_out[l + 1] - s_out[l]);
      const size_t o = axis == 0 ? static_cast<size_t>(l) * W + line
                                 : static_cast<size_t>(line) * (W - 1) + l;
      d_f[o] = df;
      vv[o] = fmax(0.0, df - db);
    }
  }
}

// numpy pairwise summation (pairwise_sum in loops_utils.h): blocks of <=128
// elements with 8 accumulators, recursive halving at multiples of 8.
__device__ double pairwise_leaf(const double* a, long long n) {
  if (n < 8) {
    double r = 0.0;
    for (long long i = 0; i < n; ++i) r = r + a[i];
    return r;
  }
  double r[8];
  for (int k = 0; k < 8; ++k) r[k] = a[k];
  long long i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int k = 0; k < 8; ++k) r[k] = r[k] + a[i + k];
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res = res + a[i];
  return res;
}

// the recursion tree is fixed by n: leaves are evaluated in parallel, then
// combined bottom-up in the recursion's pairing order by one thread
struct PwNode {
  long long off, n;
  int left, right;  // children, -1 for a leaf
  double val;
};


// blurriness (:310-332): scores (s_f - v.sum()) / s_f per axis with s_f > 0
__global__ void k_blur_finish(const double* sums, int n_axes, double* blur_weight) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  bool any = false;
  double best = 0.0;
  for (int a = 0; a < n_axes; ++a) {
    const double s_f = sums[2 * a], s_v = sums[2 * a + 1];
    if (s_f > 0) {
      const double sc = (s_f - s_v) / s_f;
      if (!any || sc > best) best = sc;  // Python max(): first maximum wins
      any = true;
    }
  }
  if (!any) {
    *blur_weight = 1.0;
    return;
  }
  *blur_weight = fmin(fmax(1.0 - best, 0.0), 1.0);
}

// ---------------------------------------------------------------------------
// fuse_color (:377-460)

constexpr int kMaxMembers = 64;

struct MemberDev {
  const double* depth;
  const double* w_map;
  const double* color;
  const double* blur;
  rf_pose rel;
};

// The member table travels as a kernel parameter (8 KB; no host->device
// copy that would wait for the stream).
struct MemberTable {
  MemberDev m[kMaxMembers];
};

__device__ __forceinline__ void bilinear(const double* img, int W, int H, double u, double v,
                                         double out[3]) {  // _bilinear (:362-374)
  long long u0 = static_cast<long long>(floor(u)), v0 = static_cast<long long>(floor(v));
  u0 = min(max(u0, 0LL), static_cast<long long>(W - 1));
  v0 = min(max(v0, 0LL), static_cast<long long>(H - 1));
  const long long u1 = min(u0 + 1, static_cast<long long>(W - 1));
  const long long v1 = min(v0 + 1, static_cast<long long>(H - 1));
  const double fu = u - static_cast<double>(u0), fv = v - static_cast<double>(v0);
  for (int c = 0; c < 3; ++c) {
    const double a = img[(v0 * W + u0) * 3 + c], b = img[(v0 * W + u1) * 3 + c];
    const double d = img[(v1 * W + u0) * 3 + c], e = img[(v1 * W + u1) * 3 + c];
    const double top = a * (1 - fu) + b * fu;
    const double bot = d * (1 - fu) + e * fu;
    out[c] = top * (1 - fv) + bot * fv;
  }
}

__global__ void k_fuse_color(const double* __restrict__ kd, const double* __restrict__ kw, Intr in,
                             const __grid_constant__ MemberTable tab, int n_mem, double delta_occl,
                             int order, double* __restrict__ color_out,
                             unsigned char* __restrict__ valid_out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= in.w * in.h) return;
  double* co = color_out + 3 * static_cast<size_t>(i);
  co[0] = co[1] = co[2] = 0.0;
  valid_out[i] = 0;
  if (!(kw[i] > 0.0)) return;
  const int u = i % in.w, v = i / in.w;
  const double z = kd[i];
  const double p0 = ((static_cast<double>(u) - in.cx) / in.fx) * z;
  const double p1 = ((static_cast<double>(v) - in.cy) / in.fy) * z;
  double vals[kMaxMembers][3];
  double wts[kMaxMembers];
  for (int m = 0; m < n_mem; ++m) {
    vals[m][0] = vals[m][1] = vals[m][2] = 0.0;
    wts[m] = 0.0;
    const MemberDev& M = tab.m[m];
    double q0, q1, q2;
    transform(M.rel, p0, p1, z, order, q0, q1, q2);
    if (!(q2 > 0)) continue;
    const double uu = in.fx * q0 / q2 + in.cx;
    const double vv = in.fy * q1 / q2 + in.cy;
    if (!(uu >= 0 && uu <= in.w - 1 && vv >= 0 && vv <= in.h - 1)) continue;
    const int un = static_cast<int>(floor(uu + 0.5)), vn = static_cast<int>(floor(vv + 0.5));
    const size_t q = static_cast<size_t>(vn) * in.w + un;
    const double zn = M.depth[q];
    const double w_c = *M.blur * M.w_map[q];
    if (!(zn > 0 && fabs(zn - q2) <= delta_occl && w_c > 0)) continue;
    bilinear(M.color, in.w, in.h, uu, vv, vals[m]);
    wts[m] = w_c;
  }
  double total = 0.0;
  for (int m = 0; m < n_mem; ++m) total = total + wts[m];  // sum(axis=0)
  if (!(total > 0)) return;
  const double half = total / 2.0;
  int idx[kMaxMembers];
  for (int ch = 0; ch < 3; ++ch) {
    for (int m = 0; m < n_mem; ++m) idx[m] = m;
    for (int a = 1; a < n_mem; ++a) {  // stable insertion sort by value
      const int key = idx[a];
      const double kv = vals[key][ch];
      int b = a - 1;
      while (b >= 0 && vals[idx[b]][ch] > kv) {
        idx[b + 1] = idx[b];
        --b;
      }
      idx[b + 1] = key;
    }
    double cum = 0.0;
    int pick = 0;  // argmax of (cum >= half): first True, else 0
    for (int a = 0; a < n_mem; ++a) {
      cum = cum + wts[idx[a]];
      if (cum >= half) {
        pick = a;
        break;
      }
    }
    co[ch] = vals[idx[pick]][ch];
  }
  valid_out[i] = 1;
}

// fuse_color with more than kMaxMembers members (KF_DIST / KF_OVRLP / KF_DVO
// keyframes that stay open, or kappa > 64): the same per-pixel semantics with
// the samples in a global scratch (one row of n_mem per pixel of a chunk) and
// a stable bottom-up merge sort instead of the insertion sort.  Zero-weight
// samples take part exactly as in the reference's argsort / cumsum (adding
// +0.0 never changes the running sum).
__global__ void k_fuse_color_big(const double* __restrict__ kd, const double* __restrict__ kw,
                                 Intr in, const MemberDev* __restrict__ tab, int n_mem,
                                 double delta_occl, int order, int p0, int count,
                                 double* __restrict__ vals, double* __restrict__ wts,
                                 int* __restrict__ idx, int* __restrict__ tmp,
                                 double* __restrict__ color_out,
                                 unsigned char* __restrict__ valid_out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  const int i = p0 + t;
  double* co = color_out + 3 * static_cast<size_t>(i);
  co[0] = co[1] = co[2] = 0.0;
  valid_out[i] = 0;
  if (!(kw[i] > 0.0)) return;
  double* V = vals + static_cast<size_t>(t) * n_mem * 3;
  double* Wt = wts + static_cast<size_t>(t) * n_mem;
  int* I = idx + static_cast<size_t>(t) * n_mem;
  int* Tm = tmp + static_cast<size_t>(t) * n_mem;
  const int u = i % in.w, v = i / in.w;
  const double z = kd[i];
  const double p0x = ((static_cast<double>(u) - in.cx) / in.fx) * z;
  const double p1x = ((static_cast<double>(v) - in.cy) / in.fy) * z;
  for (int m = 0; m < n_mem; ++m) {
    double c3[3] = {0.0, 0.0, 0.0};
    double wc = 0.0;
    const MemberDev& M = tab[m];
    double q0, q1, q2;
    transform(M.rel, p0x, p1x, z, order, q0, q1, q2);
    if (q2 > 0) {
      const double uu = in.fx * q0 / q2 + in.cx;
      const double vv = in.fy * q1 / q2 + in.cy;
      if (uu >= 0 && uu <= in.w - 1 && vv >= 0 && vv <= in.h - 1) {
        const int un = static_cast<int>(floor(uu + 0.5)), vn = static_cast<int>(floor(vv + 0.5));
        const size_t q = static_cast<size_t>(vn) * in.w + un;
        const double zn = M.depth[q];
        const double w_c = *M.blur * M.w_map[q];
        if (zn > 0 && fabs(zn - q2) <= delta_occl && w_c > 0) {
          bilinear(M.color, in.w, in.h, uu, vv, c3);
          wc = w_c;
        }
      }
    }
    V[3 * m] = c3[0];
    V[3 * m + 1] = c3[1];
    V[3 * m + 2] = c3[2];
    Wt[m] = wc;
  }
  double total = 0.0;
  for (int m = 0; m < n_mem; ++m) total = total + Wt[m];
  if (!(total > 0)) return;
  const double half = total / 2.0;
  for (int ch = 0; ch < 3; ++ch) {
    for (int m = 0; m < n_mem; ++m) I[m] = m;
    // stable bottom-up merge sort of I by V[.][ch]
    int* src = I;
    int* dst = Tm;
    for (int width = 1; width < n_mem; width *= 2) {
      for (int lo = 0; lo < n_mem; lo += 2 * width) {
        const int mid = min(lo + width, n_mem), hi = min(lo + 2 * width, n_mem);
        int a = lo, b = mid, o = lo;
        while (a < mid && b < hi) {
          // take from the right run only when strictly smaller: stable
          if (V[3 * src[b] + ch] < V[3 * src[a] + ch]) dst[o++] = src[b++];
          else dst[o++] = src[a++];
        }
        while (a < mid) dst[o++] = src[a++];
        while (b < hi) dst[o++] = src[b++];
      }
      int* sw = src;
      src = dst;
      dst = sw;
    }
    double cum = 0.0;
    int pick = 0;
    for (int a = 0; a < n_mem; ++a) {
      cum = cum + Wt[src[a]];
      if (cum >= half) {
        pick = a;
        break;
      }
    }
    co[ch] = V[3 * src[pick] + ch];
  }
  valid_out[i] = 1;
}

Intr make_intr(int w, int h, double fx, double fy, double cx, double cy) {
  Intr in;
  in.w = w;
  in.h = h;
  in.fx = fx;
  in.fy = fy;
  in.cx = cx;
  in.cy = cy;
  return in;
}

int build_pairwise_tree(long long off, long long n, std::vector<PwNode>& out) {
  if (n <= 128) {
    out.push_back({off, n, -1, -1, 0.0});
    return static_cast<int>(out.size()) - 1;
  }
  long long n2 = n / 2;
  n2 -= n2 % 8;
  const int l = build_pairwise_tree(off, n2, out);
  const int r = build_pairwise_tree(off + n2, n - n2, out);
  out.push_back({off, n, l, r, 0.0});
  return static_cast<int>(out.size()) - 1;
}

// numpy's pairwise tree for n elements, sorted by height and uploaded once
// per (device, n): [leaves | height-1 nodes | ...], children before parents.
struct PwTree {
  PwNode* nodes = nullptr;
  int* level_off = nullptr;
  int n_nodes = 0, n_leaves = 0, n_levels = 0;
};

const PwTree* pairwise_tree(long long n) {
  static std::map<std::pair<int, long long>, PwTree> cache;
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find({dev, n});
  if (it != cache.end()) return &it->second;
  std::vector<PwNode> post;
  build_pairwise_tree(0, n, post);
  const int m = static_cast<int>(post.size());
  std::vector<int> height(m, 0);
  int max_h = 0;
  for (int k = 0; k < m; ++k)  // post-order: children first
    if (post[k].left >= 0) {
      height[k] = std::max(height[post[k].left], height[post[k].right]) + 1;
      max_h = std::max(max_h, height[k]);
    }
  std::vector<int> order(m), pos(m), level_off(max_h + 2, 0);
  for (int k = 0; k < m; ++k) ++level_off[height[k] + 1];
  for (int h = 0; h <= max_h; ++h) level_off[h + 1] += level_off[h];
  std::vector<int> fill(level_off.begin(), level_off.end() - 1);
  for (int k = 0; k < m; ++k) pos[k] = fill[height[k]]++;  // stable within a level
  std::vector<PwNode> sorted(m);
  for (int k = 0; k < m; ++k) {
    PwNode e = post[k];
    if (e.left >= 0) {
      e.left = pos[e.left];
      e.right = pos[e.right];
    }
    sorted[pos[k]] = e;
  }
  PwTree t;
  t.n_nodes = m;
  t.n_leaves = level_off[1];
  t.n_levels = max_h + 1;
  if (cudaMalloc(&t.nodes, sizeof(PwNode) * m) != cudaSuccess ||
      cudaMalloc(&t.level_off, sizeof(int) * level_off.size()) != cudaSuccess)
    return nullptr;
  cudaMemcpy(t.nodes, sorted.data(), sizeof(PwNode) * m, cudaMemcpyHostToDevice);
  cudaMemcpy(t.level_off, level_off.data(), sizeof(int) * level_off.size(), cudaMemcpyHostToDevice);
  return &cache.emplace(std::make_pair(dev, n), t).first->second;
}

// Up to four pairwise sums at once: leaves of all trees in one grid, then
// one CTA per tree for the levels.
struct PwBatch {
  const double* a[4];
  const PwNode* nodes[4];
  const int* level_off[4];
  double* val[4];
  double* out[4];
  int n_leaves[4], n_levels[4], leaf_base[5];
};

__global__ void k_pairwise_leaves_batch(PwBatch b) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  int t = 0;
  while (t < 3 && k >= b.leaf_base[t + 1]) ++t;
  const int j = k - b.leaf_base[t];
  if (k >= b.leaf_base[4] || j >= b.n_leaves[t]) return;
  b.val[t][j] = pairwise_leaf(b.a[t] + b.nodes[t][j].off, b.nodes[t][j].n);
}

__global__ void __launch_bounds__(1024) k_pairwise_levels_batch(PwBatch b) {
  const int t = blockIdx.x;
  const PwNode* nodes = b.nodes[t];
  const int* lo = b.level_off[t];
  double* val = b.val[t];
  for (int l = 1; l < b.n_levels[t]; ++l) {
    for (int k = lo[l] + threadIdx.x; k < lo[l + 1]; k += blockDim.x)
      val[k] = val[nodes[k].left] + val[nodes[k].right];
    __syncthreads();
  }
  if (threadIdx.x == 0) *b.out[t] = val[lo[b.n_levels[t]] - 1];
}

rf_status pairwise_sums(int count, const double* const* a, const long long* n, double* const* out,
                        cudaStream_t s) {
  PwBatch b{};
  double* val = nullptr;
  long long total_nodes = 0;
  const PwTree* trees[4];
  for (int t = 0; t < count; ++t) {
    trees[t] = pairwise_tree(n[t]);
    if (!trees[t]) return RF_CUDA;
    total_nodes += trees[t]->n_nodes;
  }
  if (cudaMallocAsync(&val, sizeof(double) * total_nodes, s) != cudaSuccess) return RF_CUDA;
  long long vo = 0;
  b.leaf_base[0] = 0;
  for (int t = 0; t < 4; ++t) {
    const bool on = t < count;
    b.a[t] = on ? a[t] : nullptr;
    b.nodes[t] = on ? trees[t]->nodes : nullptr;
    b.level_off[t] = on ? trees[t]->level_off : nullptr;
    b.val[t] = on ? val + vo : nullptr;
    b.out[t] = on ? out[t] : nullptr;
    b.n_leaves[t] = on ? trees[t]->n_leaves : 0;
    b.n_levels[t] = on ? trees[t]->n_levels : 0;
    b.leaf_base[t + 1] = b.leaf_base[t] + b.n_leaves[t];
    if (on) vo += trees[t]->n_nodes;
  }
  k_pairwise_leaves_batch<<<(b.leaf_base[4] + 127) / 128, 128, 0, s>>>(b);
  k_pairwise_levels_batch<<<count, 1024, 0, s>>>(b);
  cudaFreeAsync(val, s);
  return RF_OK;
}


// The stream-ordered pool keeps what it allocated between calls (the fusion
// entry points allocate scratch per call; releasing it at every host sync
// would re-map device memory on the next call).
void keep_pool() {
  static std::mutex mu;
  static std::vector<int> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (std::find(done.begin(), done.end(), dev) != done.end()) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    unsigned long long thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done.push_back(dev);
}

// blurriness (:310-332) of a gray image into caller scratch: b (n),
// buf (4n: d_f and v per axis), sums (4 doubles).
rf_status blurriness_core(const double* gray, int width, int height, double* b, double* buf,
                          double* sums, double* blur_weight, cudaStream_t s) {
  const long long n = static_cast<long long>(width) * height;
  // per axis: d_f and v = max(0, d_f - d_b), then the four pairwise sums at once
  const double* arr[4];
  long long cnt[4];
  double* outs[4];
  int axes = 0;
  for (int axis = 0; axis < 2; ++axis) {
    const int len = axis == 0 ? height : width;
    if (len < 2) continue;
    const int lines = axis == 0 ? width : height;
    double* d_f = buf + 2 * axes * n;
    double* vv = d_f + n;
    if (len <= kBlurMaxLen) {
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(k_blur_lines_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(sizeof(double) * 2 * kBlurMaxLen * kBlurWarps));
        attr = true;
      }
      k_blur_lines_smem<<<(lines + kBlurWarps - 1) / kBlurWarps, 32 * kBlurWarps,
                          sizeof(double) * 2 * len * kBlurWarps, s>>>(gray, width, height, axis,
                                                                     9, b, d_f, vv);
    } else {
      k_blur_lines<<<(lines + 63) / 64, 64, 0, s>>>(gray, width, height, axis, 9, b, d_f, vv);
    }
    const long long m = axis == 0 ? static_cast<long long>(height - 1) * width
                                  : static_cast<long long>(height) * (width - 1);
    arr[2 * axes] = d_f;
    arr[2 * axes + 1] = vv;
    cnt[2 * axes] = cnt[2 * axes + 1] = m;
    outs[2 * axes] = sums + 2 * axes;
    outs[2 * axes + 1] = sums + 2 * axes + 1;
    ++axes;
  }
  rf_status st = RF_OK;
  if (axes > 0 && pairwise_sums(2 * axes, arr, cnt, outs, s) != RF_OK) st = RF_CUDA;
  k_blur_finish<<<1, 1, 0, s>>>(sums, axes, blur_weight);
  return st;
}

}  // namespace

extern "C" {

rf_status rf_depth_weight(const double* depth, int32_t width, int32_t height, double fx, double fy,
                          double cx, double cy, double delta_disc, int32_t flags, double* w_map,
                          void* stream) {
  if (!depth || !w_map || width <= 0 || height <= 0) return RF_INVALID_ARG;
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  dim3 blk(32, 8), grd((width + 31) / 32, (height + 7) / 8);
  k_depth_weight<<<grd, blk, 0, s>>>(depth, make_intr(width, height, fx, fy, cx, cy), delta_disc,
                                     flags, w_map);
  return cudaGetLastError() == cudaSuccess ? RF_OK : RF_CUDA;
}

rf_status rf_fuse_depth(double* kf_depth, double* kf_weight, const double* frame_depth,
                        const double* w_map, int32_t width, int32_t height, double fx, double fy,
                        double cx, double cy, const rf_pose* rel, int32_t blas_order,
                        void* stream) {
  if (!kf_depth || !kf_weight || !frame_depth || !w_map || !rel || width <= 0 || height <= 0 ||
      static_cast<long long>(width) * height >= (1LL << 30))
    return RF_INVALID_ARG;
  keep_pool();
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int n = width * height;
  // one scratch allocation: ints [target | counts | cursor | offsets | slots],
  // doubles [val_wz | val_w], then the scan's temporary storage
  size_t scan_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, static_cast<const int*>(nullptr),
                                static_cast<int*>(nullptr), n, s);
  const size_t off_d = (sizeof(int) * 5 * static_cast<size_t>(n) + 255) & ~size_t(255);
  const size_t off_scan = (off_d + sizeof(double) * 2 * static_cast<size_t>(n) + 255) & ~size_t(255);
  char* mem = nullptr;
  if (cudaMallocAsync(&mem, off_scan + scan_bytes, s) != cudaSuccess) return RF_CUDA;
  int* target = reinterpret_cast<int*>(mem);
  int* counts = target + n;
  int* cursor = counts + n;
  int* offsets = cursor + n;
  int* slots = offsets + n;
  double* vwz = reinterpret_cast<double*>(mem + off_d);
  double* vw = vwz + n;
  cudaMemsetAsync(counts, 0, sizeof(int) * 2 * n, s);  // counts + cursor
  const Intr in = make_intr(width, height, fx, fy, cx, cy);
  k_warp<<<(n + 255) / 256, 256, 0, s>>>(frame_depth, w_map, in, *rel, blas_order, target, vwz, vw,
                                          counts);
  cub::DeviceScan::ExclusiveSum(mem + off_scan, scan_bytes, counts, offsets, n, s);
  k_scatter<<<(n + 255) / 256, 256, 0, s>>>(target, n, offsets, cursor, slots);
  k_merge<<<(n + 255) / 256, 256, 0, s>>>(kf_depth, kf_weight, n, counts, offsets, slots, vwz, vw);
  cudaFreeAsync(mem, s);
  return cudaGetLastError() == cudaSuccess ? RF_OK : RF_CUDA;
}

rf_status rf_fuse_frame(double* kf_depth, double* kf_weight, const double* frame_depth,
                        const double* frame_color, int32_t width, int32_t height, double fx,
                        double fy, double cx, double cy, const rf_pose* rel, int32_t blas_order,
                        double delta_disc, const double* gauss_weights, int32_t radius,
                        double gain, double* w_map, double* depth_copy, double* member_color,
                        double* blur_weight, void* stream) {
  if (!kf_depth || !kf_weight || !frame_depth || !rel || !w_map || !depth_copy ||
      width <= 0 || height <= 0 || static_cast<long long>(width) * height >= (1LL << 30))
    return RF_INVALID_ARG;
  if (frame_color && (!member_color || !blur_weight || !gauss_weights || radius < 0 ||
                      radius > 15))
    return RF_INVALID_ARG;
  keep_pool();
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int n = width * height;
  // one scratch allocation: ints [target | counts | cursor | offsets | slots],
  // doubles [val_wz | val_w | gray | gauss tmp (3n) | blur b | blur buf (4n) | sums]
  size_t scan_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, static_cast<const int*>(nullptr),
                                static_cast<int*>(nullptr), n, s);
  const size_t ints = 5 * static_cast<size_t>(n);
  const size_t dbl = (frame_color ? 11 : 2) * static_cast<size_t>(n) + 4;
  const size_t off_d = (sizeof(int) * ints + 255) & ~size_t(255);
  const size_t off_scan = (off_d + sizeof(double) * dbl + 255) & ~size_t(255);
  char* mem = nullptr;
  if (cudaMallocAsync(&mem, off_scan + scan_bytes, s) != cudaSuccess) return RF_CUDA;
  int* target = reinterpret_cast<int*>(mem);
  int* counts = target + n;
  int* cursor = counts + n;
  int* offsets = cursor + n;
  int* slots = offsets + n;
  double* vwz = reinterpret_cast<double*>(mem + off_d);
  double* vw = vwz + n;
  const Intr in = make_intr(width, height, fx, fy, cx, cy);
  cudaMemsetAsync(counts, 0, sizeof(int) * 2 * n, s);  // counts + cursor
  const dim3 blk(32, 8), grd((width + 31) / 32, (height + 7) / 8);
  k_dw_warp<<<grd, blk, 0, s>>>(frame_depth, in, delta_disc, *rel, blas_order, w_map, depth_copy,
                                target, vwz, vw, counts);
  cub::DeviceScan::ExclusiveSum(mem + off_scan, scan_bytes, counts, offsets, n, s);
  k_scatter<<<(n + 255) / 256, 256, 0, s>>>(target, n, offsets, cursor, slots);
  k_merge<<<(n + 255) / 256, 256, 0, s>>>(kf_depth, kf_weight, n, counts, offsets, slots, vwz, vw);
  rf_status st = RF_OK;
  if (frame_color) {  // colour prep (:278-281): unsharp mask + blurriness of grayscale
    double* gray = vw + n;
    double* gtmp = gray + n;
    double* bb = gtmp + 3 * static_cast<size_t>(n);
    double* bbuf = bb + n;
    double* sums = bbuf + 4 * static_cast<size_t>(n);
    GaussW g;
    g.r = radius;
    for (int j = 0; j <= radius; ++j) g.w[j] = gauss_weights[radius + j];  // symmetric
    k_gauss_rows_gray<<<grd, blk, 0, s>>>(frame_color, width, height, g, gtmp, gray);
    if (gain == 0.0)  // unsharp_mask returns img.copy() (:338-339)
      cudaMemcpyAsync(member_color, frame_color, sizeof(double) * 3 * n,
                      cudaMemcpyDeviceToDevice, s);
    else
      k_gauss_cols_unsharp<<<grd, blk, 0, s>>>(frame_color, gtmp, width, height, 3, g, gain,
                                               member_color);
    st = blurriness_core(gray, width, height, bb, bbuf, sums, blur_weight, s);
  }
  cudaFreeAsync(mem, s);
  if (st != RF_OK) return st;
  return cudaGetLastError() == cudaSuccess ? RF_OK : RF_CUDA;
}

rf_status rf_unsharp_mask(const double* img, int32_t width, int32_t height, int32_t channels,
                          const double* gauss_weights, int32_t radius, double gain, double* out,
                          void* stream) {
  if (!img || !out || !gauss_weights || width <= 0 || height <= 0 || channels <= 0 ||
      radius < 0 || radius > 15)
    return RF_INVALID_ARG;
  keep_pool();
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long long n = static_cast<long long>(width) * height * channels;
  if (gain == 0.0) {  // unsharp_mask returns img.copy() (:338-339)
    cudaMemcpyAsync(out, img, sizeof(double) * n, cudaMemcpyDeviceToDevice, s);
    return cudaGetLastError() == cudaSuccess ? RF_OK : RF_CUDA;
  }
  GaussW g;
  g.r = radius;
  for (int j = 0; j <= radius; ++j) g.w[j] = gauss_weights[radius + j];  // symmetric
  double* tmp = nullptr;
  if (cudaMallocAsync(&tmp, sizeof(double) * n, s) != cudaSuccess) return RF_CUDA;
  dim3 blk(32, 8), grd((width + 31) / 32, (height + 7) / 8);
  k_gauss_rows<<<grd, blk, 0, s>>>(img, width, height, channels, g, tmp);
  k_gauss_cols_unsharp<<<grd, blk, 0, s>>>(img, tmp, width, height, channels, g, gain, out);
  cudaFreeAsync(tmp, s);
  return cudaGetLastError() == cudaSuccess ? RF_OK : RF_CUDA;
}

rf_status rf_grayscale(const double* color, int32_t width, int32_t height, double* gray,
                       void* stream) {
  if (!color || !gray || width <= 0 || height <= 0) return RF_INVALID_ARG;
  const int n = width * height;
  k_gray<<<(n + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(color, n, gray);
  return cudaGetLastError() == cudaSuccess ? RF_OK : RF_CUDA;
}

rf_status rf_blurriness(const double* gray, int32_t width, int32_t height, double* blur_weight,
                        void* stream) {
  if (!gray || !blur_weight || width <= 0 || height <= 0) return RF_INVALID_ARG;
  keep_pool();
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long long n = static_cast<long long>(width) * height;
  double* scratch = nullptr;
  if (cudaMallocAsync(&scratch, sizeof(double) * (5 * n + 4), s) != cudaSuccess) return RF_CUDA;
  const rf_status st = blurriness_core(gray, width, height, scratch, scratch + n,
                                       scratch + 5 * n, blur_weight, s);
  cudaFreeAsync(scratch, s);
  if (st != RF_OK) return st;
  return cudaGetLastError() == cudaSuccess ? RF_OK : RF_CUDA;
}

rf_status rf_color_prep(const double* color, int32_t width, int32_t height,
                        const double* gauss_weights, int32_t radius, double gain,
                        double* member_color, double* blur_weight, void* stream) {
  if (!color || !member_color || !blur_weight) return RF_INVALID_ARG;
  keep_pool();
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* gray = nullptr;
  if (cudaMallocAsync(&gray, sizeof(double) * width * height, s) != cudaSuccess) return RF_CUDA;
  rf_status st = rf_unsharp_mask(color, width, height, 3, gauss_weights, radius, gain,
                                 member_color, stream);
  if (st == RF_OK) st = rf_grayscale(color, width, height, gray, stream);
  if (st == RF_OK) st = rf_blurriness(gray, width, height, blur_weight, stream);
  cudaFreeAsync(gray, s);
  return st;
}

rf_status rf_fuse_color(const double* kf_depth, const double* kf_weight, int32_t width,
                        int32_t height, double fx, double fy, double cx, double cy,
                        int32_t n_members, const rf_member_view* members, double delta_occl,
                        int32_t blas_order, double* kf_color, uint8_t* color_valid,
                        void* stream) {
  if (!kf_depth || !kf_weight || !kf_color || !color_valid || width <= 0 || height <= 0 ||
      n_members < 0 || (n_members > 0 && !members))
    return RF_INVALID_ARG;
  keep_pool();
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<MemberDev> host(static_cast<size_t>(std::max(n_members, 1)));
  for (int m = 0; m < n_members; ++m) {
    if (!members[m].depth || !members[m].w_map || !members[m].color || !members[m].blur_weight)
      return RF_INVALID_ARG;
    host[m].depth = members[m].depth;
    host[m].w_map = members[m].w_map;
    host[m].color = members[m].color;
    host[m].blur = members[m].blur_weight;
    host[m].rel = members[m].rel;
  }
  const int n = width * height;
  if (n_members > kMaxMembers) {  // rare: global-scratch path, pixel chunks
    const Intr in = make_intr(width, height, fx, fy, cx, cy);
    const size_t per = static_cast<size_t>(n_members) * (4 * sizeof(double) + 2 * sizeof(int));
    const int chunk = static_cast<int>(std::max<size_t>(
        1, std::min<size_t>(n, (size_t(256) << 20) / per)));
    char* scratch = nullptr;
    MemberDev* d_tab = nullptr;
    if (cudaMallocAsync(&scratch, per * chunk, s) != cudaSuccess ||
        cudaMallocAsync(&d_tab, sizeof(MemberDev) * n_members, s) != cudaSuccess)
      return RF_CAPACITY;
    cudaMemcpyAsync(d_tab, host.data(), sizeof(MemberDev) * n_members, cudaMemcpyHostToDevice, s);
    double* vals = reinterpret_cast<double*>(scratch);
    double* wts = vals + static_cast<size_t>(chunk) * n_members * 3;
    int* idx = reinterpret_cast<int*>(wts + static_cast<size_t>(chunk) * n_members);
    int* tmp = idx + static_cast<size_t>(chunk) * n_members;
    for (int p0 = 0; p0 < n; p0 += chunk) {
      const int cnt = std::min(chunk, n - p0);
      k_fuse_color_big<<<(cnt + 127) / 128, 128, 0, s>>>(kf_depth, kf_weight, in, d_tab,
                                                          n_members, delta_occl, blas_order, p0,
                                                          cnt, vals, wts, idx, tmp, kf_color,
                                                          color_valid);
    }
    cudaFreeAsync(d_tab, s);
    cudaFreeAsync(scratch, s);
    // the pageable table copy above completed before returning (host order)
    return cudaGetLastError() == cudaSuccess ? RF_OK : RF_CUDA;
  }
  MemberTable tab{};
  for (int m = 0; m < n_members; ++m) tab.m[m] = host[m];
  k_fuse_color<<<(n + 127) / 128, 128, 0, s>>>(kf_depth, kf_weight,
                                                make_intr(width, height, fx, fy, cx, cy), tab,
                                                n_members, delta_occl, blas_order, kf_color,
                                                color_valid);
  return cudaGetLastError() == cudaSuccess ? RF_OK : RF_CUDA;
}

rf_status rf_normal_map(const double* depth, int32_t width, int32_t height, double fx,
                        double fy, double cx, double cy, double* normals, void* stream) {
  if (!depth || !normals || width <= 0 || height <= 0) return RF_INVALID_ARG;
  const dim3 blk(32, 8), grd((width + 31) / 32, (height + 7) / 8);
  k_normal_map<<<grd, blk, 0, static_cast<cudaStream_t>(stream)>>>(
      depth, make_intr(width, height, fx, fy, cx, cy), normals);
  return cudaGetLastError() == cudaSuccess ? RF_OK : RF_CUDA;
}

rf_status rf_depth_sample_weight_normals(const double* depth, const double* normals,
                                         int32_t width, int32_t height, double fx, double fy,
                                         double cx, double cy, double* w, void* stream) {
  if (!depth || !normals || !w || width <= 0 || height <= 0) return RF_INVALID_ARG;
  const dim3 blk(32, 8), grd((width + 31) / 32, (height + 7) / 8);
  k_weight_from_normals<<<grd, blk, 0, static_cast<cudaStream_t>(stream)>>>(
      depth, normals, make_intr(width, height, fx, fy, cx, cy), w);
  return cudaGetLastError() == cudaSuccess ? RF_OK : RF_CUDA;
}

}  // extern "C"
