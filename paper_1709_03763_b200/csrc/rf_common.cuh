// rf_common.cuh -- shared device definitions of the B200 surface-correction path.
//
// Layout in HBM:
//   heads[hash_buckets]  int32   bucket -> first node (slot) or -1
//   keys[capacity]       int64   packed block key per slot, -1 when free
//   next[capacity]       int32   overflow linked list
//   nz[capacity]         int32   number of voxels with W != 0 (GC without scanning W)
//   stamp[capacity]      uint32  last op epoch that touched the slot (dedupe)
//   pool[capacity][5][512] f64   D, W, C0, C1, C2 planes per 8^3 block
// Slot i is hash node i and pool block i.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rf {

constexpr int kBlockSide = 8;
constexpr int kBlockVoxels = 512;
constexpr int kBlockDoubles = 5 * kBlockVoxels;
constexpr long long kPackBias = 1LL << 20;
constexpr long long kPackMask = (1LL << 21) - 1;
constexpr long long kNoKey = 0x7fffffffffffffffLL;
constexpr unsigned kFull = 0xffffffffu;
constexpr int kFuseThreads = 256;
// touched-list entry: slot | kNewFlag (the op created the block: all zero)
constexpr unsigned kNewFlag = 0x80000000u;
constexpr unsigned kSlotMask = 0x3fffffffu;

enum ErrKind : int { kErrNone = 0, kErrContract = 1, kErrInconsistent = 2, kErrCapacity = 3 };

// volume.py:137-141
__host__ __device__ __forceinline__ long long pack_key(long long bx, long long by, long long bz) {
  return ((bx + kPackBias) << 42) | ((by + kPackBias) << 21) | (bz + kPackBias);
}

// volume.py:144-148
__host__ __device__ __forceinline__ void unpack_key(long long k, long long& bx, long long& by,
                                                    long long& bz) {
  bz = (k & kPackMask) - kPackBias;
  by = ((k >> 21) & kPackMask) - kPackBias;
  bx = (k >> 42) - kPackBias;
}

// volume.py:84-93 -- Python's floor-mod of the XOR of prime products.
__host__ __device__ __forceinline__ long long block_hash(long long x, long long y, long long z,
                                                         long long buckets) {
  long long h = (x * 73856093LL) ^ (y * 19349669LL) ^ (z * 83492791LL);
  long long r = h % buckets;
  return r < 0 ? r + buckets : r;
}

__host__ __device__ __forceinline__ long long block_hash_of_key(long long key, long long buckets) {
  long long bx, by, bz;
  unpack_key(key, bx, by, bz);
  return block_hash(bx, by, bz, buckets);
}

// Shard ownership: a 64-bit finaliser independent of block_hash's low bits,
// so every shard's bucket array is loaded uniformly.
__host__ __device__ __forceinline__ int key_owner(long long key, int shards) {
  unsigned long long z = static_cast<unsigned long long>(key) + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return static_cast<int>(z % static_cast<unsigned long long>(shards));
}

// Per-op counters; one record per device op of a window (stream or
// (de)integration), reset by k_reset_ops at window start.
struct OpCounters {
  unsigned long long n_touched;       // footprint blocks (deduped)
  unsigned long long n_new;           // blocks created by this op
  unsigned long long voxels_updated;  // integrate count (fuse_block returns)
  unsigned long long streamed_in;     // stream ops
  unsigned long long streamed_out;
  unsigned long long n_pending;       // distinct missing keys found by k_footprint
  unsigned long long n_spill;         // tile keys that overflowed shared memory
  unsigned long long kf_hash;         // content hash of the op's keyframe (memo guard)
  int use_full;                       // 1: the full footprint kernel must run
  long long viol_key;                 // min footprint key outside the sphere (contract)
  long long fail_key;                 // min key whose removal check failed
  int executed;                       // 1 once the op's first kernel ran
  int capacity;                       // 1 when the pool overflowed
  // voxels a fuse kernel defers to its exact IEEE tail (operands outside
  // the fast paths' exponent range), and the kernel's finished-CTA count;
  // index 0 the removal check, 1 integrate / removal, 2 the fix-up
  unsigned n_defer[3];
  unsigned done_ctas[3];
  unsigned capture_n;  // sharded footprint: memo keys written so far
  unsigned next_block[3];  // fuse kernels: dynamic block queue (per defer index)
  unsigned fp_done;        // footprint kernel: finished CTAs
};

// Allocator state (device).  Pops during one footprint kernel only read the
// free stack; the next kernel of the op folds pops and loser returns back.
struct AllocState {
  int free_top;            // valid entries in free_stack
  int hwm;                 // slots [0, hwm) have been handed out at least once
  unsigned int pop_count;  // pops from the free stack since the last fix-up
  unsigned int n_returned; // slots returned by losing inserts since the last fix-up
  long long n_live;        // live blocks
  unsigned long long total_streamed_in;
  unsigned long long total_streamed_out;
};

// Sticky window error: ops after err_op become no-ops.
struct WinState {
  int err_kind;
  int err_op;
};

struct Table {
  int* heads;
  long long* keys;
  int* next;
  int* nz;
  unsigned* stamp;
  double* pool;
  int* free_stack;
  int* returned;
  int* touched;   // slot | kNewFlag
  int* tpos;      // per slot: its index in the current touched list
  long long* touched_keys;  // packed key of touched[i] (fuse reads no keys[] indirection)
  int* new_list;  // slots created by the current op
  long long* pend_tab;   // open-addressing set of keys to create (-1 = empty)
  long long* pend_keys;  // distinct pending keys of the current op
  int* pend_idx;         // their pend_tab index
  int pend_mask;         // pend_tab size - 1 (power of two)
  long long* spill_keys; // tile keys that did not fit in shared memory
  int spill_cap;
  AllocState* alloc;
  unsigned long long* defer;  // deferred voxels: slot << 10 | fresh << 9 | voxel
  int defer_cap;
  long long buckets;
  int capacity;
};

struct KfView {
  const double* depth;
  const double* weight;
  const double* color;  // may be null
  int width, height;
  double fx, fy, cx, cy;
};

// Programmatic dependent launch (sm_90+): batch kernels are launched with
// programmatic stream serialization, so a kernel's CTAs are scheduled while
// its predecessor drains; each waits here before reading anything the
// predecessor (or, transitively, earlier work) produced.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ bool ws_skip(const WinState* ws, int op_index) {
  const int kind = *reinterpret_cast<const volatile int*>(&ws->err_kind);
  return kind != kErrNone && *reinterpret_cast<const volatile int*>(&ws->err_op) < op_index;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ||centre(b) - c||^2 summed as volume.py:345-346 does, (dx^2 + dy^2) + dz^2.
// The reference compares sqrt of it with stream_radius; since the IEEE
// square root is monotone, sqrt(x) <= R  <=>  x <= radius2 with radius2 the
// largest double whose square root rounds to <= R (sqrt_le_bound, host),
// so the kernels compare squared distances and never take a square root.

__host__ __device__ __forceinline__ double block_center_dist2_free(long long key, double span,
                                                          const double* c) {
  long long bx, by, bz;
  unpack_key(key, bx, by, bz);
  const double dx = (static_cast<double>(bx) + 0.5) * span - c[0];
  const double dy = (static_cast<double>(by) + 0.5) * span - c[1];
  const double dz = (static_cast<double>(bz) + 0.5) * span - c[2];
  return dx * dx + dy * dy + dz * dz;
}

}  // namespace rf
