// rf_fuse_legacy.cuh -- the previous fuse kernel (CTA per block, 8 warps on
// its 8 z-slices, TMA bulk L2 prefetch of the next block's planes, plain
// predicated loads), kept as an A/B baseline for the pipelined k_fuse
// (select with RF_FUSE_IMPL=legacy).  Same arithmetic contract.
#pragma once

#include "rf_kernels.cuh"

namespace rf {

constexpr int kLegacyVoxPerLane = 2;

// Per-lane voxel-centre offsets (l_axis + 0.5) * voxel_size, computed once
// (the same rounded products as _kernels_cy.pyx:55-57).
struct LegacyLaneOffsets {
  double hx, hy[2];
};

__device__ __forceinline__ LegacyLaneOffsets legacy_lane_offsets(double vs) {
  const int lane = threadIdx.x & 31;
  LegacyLaneOffsets o;
  o.hx = (static_cast<double>(lane & 7) + 0.5) * vs;
  o.hy[0] = (static_cast<double>(lane >> 3) + 0.5) * vs;
  o.hy[1] = (static_cast<double>((lane >> 3) + 4) + 0.5) * vs;
  return o;
}

// Fuse one 64-voxel slice of a block with one warp (fuse_block's per-voxel
// update, _kernels_cy.pyx:51-105): lane handles voxels (x = lane&7,
// y = lane>>3 + 4k, z = slice), k = 0, 1.  The code is straight-line:
// every lane computes, loads and stores are predicated on the band test,
// and the only branch is the (never-taken in practice) exact-division
// fallback.  blk: the block's 5 planes.  fresh: the block was created by
// this op, so it is all zero -- nothing is read and every voxel of the
// slice is written (recycled slots need no clearing).  kCheckRemove
// returns true when some voxel's removal would fail (no writes);
// kRemoveReadd removes then re-adds the sample (the reference's rollback of
// already-processed blocks, volume.py:331-333).
template <int kMode>
__device__ __forceinline__ bool legacy_fuse_slice(const FuseParams& p, const LegacyLaneOffsets& lo,
                                           double* __restrict__ blk, bool fresh, double ox,
                                           double oy, double oz, int slice, int& count,
                                           int& nz_delta) {
  const int lane = threadIdx.x & 31;
  const double* R = p.Rwc;
  // voxel centre - camera centre (_kernels_cy.pyx:55-60); x and z are
  // shared by the lane's two voxels, and so are the products of R's
  // columns 0 and 2 (the sums keep the reference's left-to-right order)
  const double hz = (static_cast<double>(slice) + 0.5) * p.voxel_size;
  const double dx0 = (ox + lo.hx) - p.t[0];
  const double dz0 = (oz + hz) - p.t[2];
  const double z_x = R[6] * dx0, z_z = R[8] * dz0;
  const double x_x = R[0] * dx0, x_z = R[2] * dz0;
  const double y_x = R[3] * dx0, y_z = R[5] * dz0;
  int pix[kLegacyVoxPerLane];
  double pz[kLegacyVoxPerLane];
#pragma unroll
  for (int k = 0; k < kLegacyVoxPerLane; ++k) {
    const double dy0 = (oy + lo.hy[k]) - p.t[1];
    const double z = (z_x + R[7] * dy0) + z_z;
    const double px = (x_x + R[1] * dy0) + x_z;
    const double py = (y_x + R[4] * dy0) + y_z;
    pz[k] = z;
    // uf = floor(fx * px / pz + cx + 0.5), vf likewise (:66-67)
    const double nu = p.kf.fx * px, nv = p.kf.fy * py;
    const double y = rcp_for_div(z);
    double tu = markstein(nu, z, y) + p.kf.cx + 0.5;
    double tv = markstein(nv, z, y) + p.kf.cy + 0.5;
    const bool front = z > 0.0;
    // a zero numerator of either sign gives the same floor
    const bool exact = mid400(z) && (mid400(nu) || (nu == 0.0)) && (mid400(nv) || (nv == 0.0));
    if (front && !exact) {
      tu = ieee_div(nu, z) + p.kf.cx + 0.5;
      tv = ieee_div(nv, z) + p.kf.cy + 0.5;
    }
    // 0 <= floor(t) < W  <=>  0 <= t < W; for t >= 0 the IEEE bit patterns
    // order like the values, so the tests and floor run on integer bits
    // (NaN fails t < W; t cannot be -0.0 here)
    const long long bu = __double_as_longlong(tu), bv = __double_as_longlong(tv);
    const bool in = front && bu >= 0 && bu < p.w_bits && bv >= 0 && bv < p.h_bits;
    pix[k] = in ? floor_nonneg(bv) * p.kf.width + floor_nonneg(bu) : -1;
  }
  // keyframe depth / weight gathers (L2-resident keyframe), band test (:72-78)
  double wk[kLegacyVoxPerLane], dd[kLegacyVoxPerLane];
  bool hit[kLegacyVoxPerLane];
#pragma unroll
  for (int k = 0; k < kLegacyVoxPerLane; ++k) {
    const bool in = pix[k] >= 0;
    const int q = in ? pix[k] : 0;
    wk[k] = in ? __ldg(&p.kf.weight[q]) : 0.0;
    const double zk = in ? __ldg(&p.kf.depth[q]) : 0.0;
    dd[k] = zk - pz[k];
  }
#pragma unroll
  for (int k = 0; k < kLegacyVoxPerLane; ++k)
    hit[k] = pix[k] >= 0 && (wk[k] > 0.0) && dd[k] <= p.mu && dd[k] >= -p.mu;
  const int base = slice * 64 + lane;
  if constexpr (kMode == kCheckRemove) {
    bool fail = false;
#pragma unroll
    for (int k = 0; k < kLegacyVoxPerLane; ++k) {
      const double wl = (hit[k] && !fresh) ? blk[kBlockVoxels + base + 32 * k] : 0.0;
      fail |= hit[k] && (wl - wk[k] < -p.eps_w);
    }
    return __any_sync(kFull, fail);
  }
  // block planes + keyframe colour, predicated on the band test
  double W0[kLegacyVoxPerLane], d[kLegacyVoxPerLane], a0[kLegacyVoxPerLane], a1[kLegacyVoxPerLane], a2[kLegacyVoxPerLane];
  double c0[kLegacyVoxPerLane], c1[kLegacyVoxPerLane], c2[kLegacyVoxPerLane];
#pragma unroll
  for (int k = 0; k < kLegacyVoxPerLane; ++k) {
    const bool ld = hit[k] && !fresh;
    const double* v = blk + base + 32 * k;
    W0[k] = ld ? v[kBlockVoxels] : 0.0;
    d[k] = ld ? v[0] : 0.0;
    a0[k] = ld ? v[2 * kBlockVoxels] : 0.0;
    a1[k] = ld ? v[3 * kBlockVoxels] : 0.0;
    a2[k] = ld ? v[4 * kBlockVoxels] : 0.0;
    const bool lc = hit[k] && p.kf.color != nullptr;
    const double* c = p.kf.color + 3 * static_cast<size_t>(lc ? pix[k] : 0);
    c0[k] = lc ? __ldg(c) : 0.0;
    c1[k] = lc ? __ldg(c + 1) : 0.0;
    c2[k] = lc ? __ldg(c + 2) : 0.0;
  }
#pragma unroll
  for (int k = 0; k < kLegacyVoxPerLane; ++k) {
    const double w = wk[k], e = dd[k];
    const double w_before = W0[k];
    double Wn = W0[k], dn = d[k], n0 = a0[k], n1 = a1[k], n2 = a2[k];
    // the four quotients of one voxel share their denominator
    auto blend = [&](double wl, double ws, double sgn) {
      // (x * wl +/- s * w) / ws for x in (d, c0, c1, c2)
      const double m0 = dn * wl + sgn * (e * w);
      const double m1 = n0 * wl + sgn * (c0[k] * w);
      const double m2 = n1 * wl + sgn * (c1[k] * w);
      const double m3 = n2 * wl + sgn * (c2[k] * w);
      const double y = rcp_for_div(ws);
      const bool exact = mid400(ws) && (mid400(m0) || pos_zero(m0)) &&
                         (mid400(m1) || pos_zero(m1)) && (mid400(m2) || pos_zero(m2)) &&
                         (mid400(m3) || pos_zero(m3));
      if (hit[k] && !exact) {
        dn = ieee_div(m0, ws);
        n0 = ieee_div(m1, ws);
        n1 = ieee_div(m2, ws);
        n2 = ieee_div(m3, ws);
      } else {
        dn = markstein(m0, ws, y);
        n0 = markstein(m1, ws, y);
        n1 = markstein(m2, ws, y);
        n2 = markstein(m3, ws, y);
      }
    };
    if (kMode == kIntegrate) {
      const double wn = Wn + w;  // :99-104
      blend(Wn, wn, 1.0);
      Wn = wn;
    } else {
      const double wn = Wn - w;  // :86-97
      if (wn < p.eps_w) {
        dn = 0.0; n0 = 0.0; n1 = 0.0; n2 = 0.0; Wn = 0.0;
      } else {
        blend(Wn, wn, -1.0);
        Wn = wn;
      }
      if (kMode == kRemoveReadd) {
        const double wa = Wn + w;
        blend(Wn, wa, 1.0);
        Wn = wa;
      }
    }
    double* v = blk + base + 32 * k;
    if (hit[k] || fresh) {
      v[0] = hit[k] ? dn : 0.0;
      v[kBlockVoxels] = hit[k] ? Wn : 0.0;
      v[2 * kBlockVoxels] = hit[k] ? n0 : 0.0;
      v[3 * kBlockVoxels] = hit[k] ? n1 : 0.0;
      v[4 * kBlockVoxels] = hit[k] ? n2 : 0.0;
    }
    if (hit[k]) {
      nz_delta += static_cast<int>(Wn != 0.0) - static_cast<int>(w_before != 0.0);
      ++count;
    }
  }
  return false;
}

// TMA bulk prefetch of touched block j's planes into L2
// (cp.async.bulk.prefetch.L2, SASS UBLKPF).  Fresh blocks are never read.
__device__ __forceinline__ void bulk_prefetch_block(const Table& T, const double* base, int j,
                                                    unsigned bytes) {
  const unsigned entry = static_cast<unsigned>(__ldg(&T.touched[j]));
  if (entry & kNewFlag) return;
  const double* src = base + static_cast<size_t>(entry & kSlotMask) * kBlockDoubles;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// Batched fuse over the op's touched list (integrate, the removal check,
// the removal, or the failed-removal fix-up).
template <int kMode>
__global__ void __launch_bounds__(kFuseThreads, kMode == kCheckRemove ? 5 : 4)
    k_fuse_legacy(Table T, FuseParams p) {
  griddep_wait();
  // the first kernel after a footprint kernel folds the allocator state
  if ((kMode == kIntegrate || kMode == kCheckRemove) && blockIdx.x == 0) alloc_fixup_cta(T);
  if (ws_skip(p.ws, p.op_index)) return;
  OpCounters* op = p.op;
  const int n = static_cast<int>(op->n_touched);
  if (kMode == kIntegrate || kMode == kCheckRemove) {
    if (op->capacity) {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        p.ws->err_kind = kErrCapacity;
        p.ws->err_op = p.op_index;
      }
      return;
    }
    if (op->viol_key != kNoKey) {
      contract_rollback(T, op, static_cast<int>(op->n_new));
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        p.ws->err_kind = kErrContract;
        p.ws->err_op = p.op_index;
      }
      return;
    }
  }
  if (kMode == kApplyRemove) {
    if (op->capacity || op->viol_key != kNoKey) return;
    if (op->fail_key != kNoKey) {  // fixed up by kRemoveReadd after the host sees it
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        p.ws->err_kind = kErrInconsistent;
        p.ws->err_op = p.op_index;
      }
      return;
    }
  }
  const long long fail_key = op->fail_key;
  if (kMode == kRemoveReadd && fail_key == kNoKey) return;
  if ((kMode == kIntegrate || kMode == kCheckRemove) && p.capture && op->use_full) {
    // memoise this op's footprint keys for the matching later op
    const int cap = p.capture->cap;
    const bool sharded = p.shard_count > 1;
    const int cnt = sharded ? static_cast<int>(op->capture_n) : n;
    if (!sharded && n <= cap) {
      for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        p.capture->keys[i] = T.keys[static_cast<unsigned>(T.touched[i]) & kSlotMask];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      p.capture->count = cnt;
      p.capture->hash = op->kf_hash;
      p.capture->valid = cnt <= cap ? 1 : 0;
    }
  }
  if (kMode == kIntegrate && p.alloc_only) {
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
      const unsigned entry = static_cast<unsigned>(T.touched[i]);
      if (!(entry & kNewFlag)) continue;
      double* blk = T.pool + static_cast<size_t>(entry & kSlotMask) * kBlockDoubles;
      for (int j = threadIdx.x; j < kBlockDoubles; j += blockDim.x) blk[j] = 0.0;
    }
    return;
  }
  const int lane = threadIdx.x & 31;
  const LegacyLaneOffsets lo = legacy_lane_offsets(p.voxel_size);
  const long long items = static_cast<long long>(n) * kSlicesPerBlock;
  const long long warps = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
  // A CTA's 8 warps take the 8 slices of one block per iteration and stride
  // by gridDim.x blocks.  Warp 0 asks the TMA unit to pull the CTA's NEXT
  // block into L2 (one bulk prefetch of its planes) while this one is fused,
  // so the per-voxel loads below hit L2 instead of waiting on HBM.
  constexpr unsigned kPrefetchBytes =
      kMode == kCheckRemove ? kBlockVoxels * 8u : static_cast<unsigned>(kBlockDoubles) * 8u;
  const double* prefetch_base = kMode == kCheckRemove ? T.pool + kBlockVoxels : T.pool;
  if (threadIdx.x == 0) {
    for (int j = blockIdx.x; j < n && j < static_cast<int>(blockIdx.x) + static_cast<int>(gridDim.x);
         j += gridDim.x)
      bulk_prefetch_block(T, prefetch_base, j, kPrefetchBytes);
  }
  int count = 0;
  for (long long it = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
       it < items; it += warps) {
    const int i = static_cast<int>(it >> 3);
    const int slice = static_cast<int>(it & 7);
    if (slice == 0 && lane == 0 && i + static_cast<int>(gridDim.x) < n)
      bulk_prefetch_block(T, prefetch_base, i + gridDim.x, kPrefetchBytes);
    const unsigned entry = static_cast<unsigned>(__ldg(&T.touched[i]));
    const int slot = static_cast<int>(entry & kSlotMask);
    const bool fresh = (entry & kNewFlag) != 0;
    const long long key = __ldg(&T.keys[slot]);
    double* blk = T.pool + static_cast<size_t>(slot) * kBlockDoubles;
    if (kMode == kRemoveReadd && key >= fail_key) {
      // the failing block and everything sorted after it stay untouched
      if (fresh)
        for (int j = lane; j < 64; j += 32)
          for (int q = 0; q < 5; ++q) blk[q * kBlockVoxels + slice * 64 + j] = 0.0;
      continue;
    }
    long long bx, by, bz;
    unpack_key(key, bx, by, bz);
    const double ox = i2d_exact(bx) * p.span;  // coord * span, volume.py:280-286
    const double oy = i2d_exact(by) * p.span;
    const double oz = i2d_exact(bz) * p.span;
    int c = 0, nzd = 0;
    const bool failed = legacy_fuse_slice<kMode>(p, lo, blk, fresh, ox, oy, oz, slice, c, nzd);
    if (kMode == kCheckRemove) {
      if (failed && lane == 0) atomicMin(&op->fail_key, key);
      continue;
    }
    count += c;
    nzd = warp_sum(nzd);
    if (lane == 0 && nzd != 0) atomicAdd(&T.nz[slot], nzd);
  }
  if (kMode == kCheckRemove) return;
  __shared__ int s_red[kFuseThreads / 32];
  const int total = block_sum<int>(count, s_red);
  if (threadIdx.x == 0 && total)
    atomicAdd(&op->voxels_updated, static_cast<unsigned long long>(total));
}

}  // namespace rf
