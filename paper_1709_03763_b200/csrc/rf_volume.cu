// rf_volume.cu -- host side of the C ABI (include/refusion_b200.h): device
// state of one sparse voxel-hashed TSDF shard and the op sequencer that turns
// the reference's volume calls into stream-ordered kernel launches.
//
// Reference behaviour followed (paths under /root/reference/pkg/src/refusion):
//   volume.py:151-197  keyframe_block_footprint  -> k_footprint
//   volume.py:216-249  allocate_blocks           -> k_footprint (+ k_fuse fix-up)
//   volume.py:296-338  integrate / deintegrate   -> k_fuse<...>
//   volume.py:341-379  stream                    -> k_stream (+ host centre/relocations)
//   volume.py:382-394  garbage_collect/total_weight
//   reintegration.py:156-223 _correct_entries    -> rf_correct (one sync per window)
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <list>
#include <unordered_map>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "refusion_b200.h"
#include "rf_kernels.cuh"
#include "rf_mesh.cuh"

#include <cub/cub.cuh>

using namespace rf;

namespace {

// entries of one rf_correct_windows call (the Python layer splits bigger
// batches at window boundaries, volume.MAX_CALL_ENTRIES)
constexpr int kMaxWindowOps = 16384;
// distinct new blocks one (de)integration may create (load factor stays low)
constexpr int kPendingSlots = 1 << 20;
// tile keys beyond a tile's shared-memory list (only pathological tiles)
constexpr int kSpillSlots = 1 << 20;
constexpr int kDeferSlots = 1 << 20;  // voxels a fuse kernel may defer to its exact tail

struct EventPair {
  cudaEvent_t a, b;
  int kind;  // 0 fuse, 1 check, 2 footprint
};

// Host index of the footprint memo: (keyframe planes, intrinsics, pose) ->
// a device FpEntry holding that footprint's keys (see rf_kernels.cuh).
struct MemoKey {
  const void* depth;
  const void* weight;
  int width, height;
  double intr[4];
  double R[9], t[3];
  bool operator==(const MemoKey& o) const { return std::memcmp(this, &o, sizeof(MemoKey)) == 0; }
};

struct MemoKeyHash {
  size_t operator()(const MemoKey& k) const {
    const unsigned char* p = reinterpret_cast<const unsigned char*>(&k);
    unsigned long long h = 1469598103934665603ull;
    for (size_t i = 0; i < sizeof(MemoKey); ++i) h = (h ^ p[i]) * 1099511628211ull;
    return static_cast<size_t>(h);
  }
};

struct MemoSlot {
  FpEntry* dev = nullptr;  // descriptor + keys: one slot of the memo arena
  int index = -1;
  std::list<MemoKey>::iterator lru;
};

}  // namespace

struct rf_volume {
  rf_config cfg{};
  cudaStream_t stream = nullptr;
  Table T{};
  OpCounters* d_ops = nullptr;
  OpCounters* h_ops = nullptr;  // pinned
  int ops_cap = 0;
  WinState* d_ws = nullptr;
  WinState* h_ws = nullptr;  // pinned
  unsigned long long* d_u64 = nullptr;  // scratch counters [8]
  unsigned long long* h_u64 = nullptr;  // pinned [8]
  double* d_wsums = nullptr;
  unsigned* d_gc_stamp = nullptr;  // per bucket: epoch of the GC that owns it
  unsigned gc_epoch = 0;
  double* d_f64 = nullptr;
  double* h_f64 = nullptr;
  AllocState* h_alloc = nullptr;  // pinned
  // host mirror of the streaming state (volume.py:104-110)
  bool has_center = false;
  double center[3] = {0, 0, 0};
  long long relocations = 0;
  unsigned epoch = 0;
  int n_sms = 148;
  int fuse_grid = 148 * 2;
  int fuse_grids[4] = {148, 148, 148, 148};  // per FuseMode, n_sms x occupancy
  int check_grid = 148;                       // k_check: n_sms x occupancy
  // staging of host keyframe planes (rf_kf_view.planes_on_host)
  struct StageSlot {
    double* buf = nullptr;
    size_t cap = 0;  // doubles
    cudaEvent_t ready = nullptr, consumed = nullptr;
    cudaEvent_t color_ready = nullptr;  // colour plane uploaded (after depth + weight)
    const void* host = nullptr;  // host depth pointer staged in this batch
    bool used = false;
    unsigned gen = 0;  // refills of this slot (its upload flags' value)
  };
  std::vector<StageSlot> stage;
  std::unordered_map<const double*, cudaEvent_t> color_ready;  // staged colour plane -> upload event
  // upload flags: per slot {depth + weight, colour}, written by the copy stream
  // after the planes (the kernels wait on them instead of the stream on events)
  unsigned* d_stage_flags = nullptr;
  size_t stage_flags_cap = 0;  // slots
  std::unordered_map<const double*, std::pair<const unsigned*, unsigned>> upload_flag;
  cudaStream_t copy_stream = nullptr;
  int stage_next = 0;
  int fp_grid_cap = 148 * 8;
  // footprint memo
  std::unordered_map<MemoKey, MemoSlot, MemoKeyHash> memo;
  std::list<MemoKey> memo_lru;
  size_t memo_budget = size_t(2) << 30;
  // fixed-size slots carved from one allocation made at first use (no
  // stream-ordered allocation inside a batch); keyframes needing more keys
  // than a slot holds are not memoised
  char* memo_arena = nullptr;
  size_t memo_slot_bytes = 0;
  int memo_slot_cap = 0;
  std::vector<int> memo_free;
  // profiling
  bool profiling = false;
  std::vector<EventPair> events;
  std::vector<cudaEvent_t> event_pool;
  long long prof_voxels = 0, prof_pixels = 0, prof_blocks = 0, prof_launches = 0;
  long long prof_int_vox = 0, prof_int_pix = 0, prof_rem_vox = 0, prof_rem_pix = 0;
  long long prof_rem_ops = 0;
  // routed footprints (hash-sharded volume, k_route): this shard's inbox and
  // every shard's (peers opened over IPC are closed on destroy)
  char* route_own = nullptr;
  char* route_peer[kMaxShards] = {};
  bool route_ipc[kMaxShards] = {};
  RouteLayout route_lay{};
  bool route_on = false;
  unsigned route_gen = 0;
  int route_nops = 0;  // ops routed by the last rf_route, consumed by the next call
  // cross-shard removal verdicts (k_shard_sync): this shard's slots, every
  // shard's (peers opened over IPC are closed on destroy)
  SyncSlot* sync_own = nullptr;
  SyncSlot* sync_peer[kMaxShards] = {};
  bool sync_ipc[kMaxShards] = {};
  // the other shards' hash tables for marching cubes' cross-shard neighbours
  // (rf_mesh_connect / rf_mesh_ipc_open); count 1 = not connected
  MeshPeers mesh{};
  void* mesh_ipc[kMaxShards][4] = {};
  int sync_max_ops = 0;
  bool sync_on = false;
  unsigned sync_gen = 0;
  std::string err;
};

namespace {

rf_status fail(rf_volume* v, rf_status st, const std::string& msg) {
  if (v) v->err = msg;
  return st;
}

#define RF_CUDA_TRY(v, expr)                                                          \
  do {                                                                                \
    cudaError_t e_ = (expr);                                                          \
    if (e_ != cudaSuccess)                                                            \
      return fail((v), RF_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));  \
  } while (0)

cudaEvent_t take_event(rf_volume* v) {
  if (!v->event_pool.empty()) {
    cudaEvent_t e = v->event_pool.back();
    v->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

struct ProfScope {
  rf_volume* v;
  int kind;
  cudaEvent_t a = nullptr;
  ProfScope(rf_volume* v_, int k) : v(v_), kind(k) {
    if (v->profiling) {
      a = take_event(v);
      cudaEventRecord(a, v->stream);
    }
  }
  ~ProfScope() {
    if (a) {
      cudaEvent_t b = take_event(v);
      cudaEventRecord(b, v->stream);
      v->events.push_back({a, b, kind});
    }
  }
};

// Largest double x with sqrt(x) <= r (IEEE sqrt, correctly rounded on host
// and device alike): the squared-distance form of `dist <= r`.
double sqrt_le_bound(double r) {
  double x = r * r;
  while (std::sqrt(x) > r) x = std::nextafter(x, 0.0);
  while (std::sqrt(std::nextafter(x, INFINITY)) <= r) x = std::nextafter(x, INFINITY);
  return x;
}

// Launch a batch kernel with programmatic stream serialization (PDL): its
// CTAs may be scheduled while the previous kernel drains; every batch kernel
// starts with griddep_wait().

template <typename... KArgs, typename... Args>
void launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
            Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

KfView to_view(const rf_kf_view* kf) {
  KfView k;
  k.depth = kf->depth;
  k.weight = kf->weight;
  k.color = kf->color;
  k.width = kf->width;
  k.height = kf->height;
  k.fx = kf->fx;
  k.fy = kf->fy;
  k.cx = kf->cx;
  k.cy = kf->cy;
  return k;
}

bool valid_kf(const rf_kf_view* kf) {
  return kf && kf->depth && kf->weight && kf->width > 0 && kf->height > 0 &&
         static_cast<long long>(kf->width) * kf->height < (1LL << 31);
}

// One batch of device ops sharing a single host synchronisation.
struct PendingStream {
  int op;
  double c[3];
  int relocated;
};

struct OpInfo {
  int kind;  // 0 stream, 1 integrate, 2 deintegrate, 3 gc, 4 allocate
  int entry;
  int window = 0;
};

struct Batch {
  rf_volume* v;
  int n_ops = 0;
  int max_ops = 0;  // op records reset by batch_begin; exceeding it is a bug
  bool has_center;
  double center[3];
  std::vector<PendingStream> streams;
  std::vector<OpInfo> infos;
  std::vector<FuseParams> fparams;  // per op (fuse ops only)
  int gc_op = -1;
  int gc_pending = -1;  // a GC op whose launch waits to be merged with the next stream op
  bool st_pending = false;  // a stream op whose scan waits to be merged into the next footprint
  StreamParams st_p{};
  // routed volume: next inbox op to consume (route_force >= 0 overrides)
  int route_next = 0;
  int route_force = -1;
};

rf_status ensure_ops(rf_volume* v, int n) {
  if (n <= v->ops_cap) return RF_OK;
  if (v->d_ops) cudaFree(v->d_ops);
  if (v->h_ops) cudaFreeHost(v->h_ops);
  v->ops_cap = std::max(n, 64);
  RF_CUDA_TRY(v, cudaMalloc(&v->d_ops, sizeof(OpCounters) * v->ops_cap));
  RF_CUDA_TRY(v, cudaMallocHost(&v->h_ops, sizeof(OpCounters) * v->ops_cap));
  return RF_OK;
}

rf_status batch_begin(rf_volume* v, Batch& b, int max_ops) {
  if (max_ops > kMaxWindowOps * 8) return fail(v, RF_INVALID_ARG, "too many ops in one call");
  rf_status st = ensure_ops(v, max_ops);
  if (st != RF_OK) return st;
  b.v = v;
  b.max_ops = std::max(max_ops, 1);
  b.has_center = v->has_center;
  std::memcpy(b.center, v->center, sizeof(b.center));
  const int n = std::max(max_ops, 1);
  {
    ProfScope ps(v, 3);
    launch(k_reset_ops, (n + 127) / 128, 128, 0, v->stream, v->d_ops, n, v->d_ws);
  }
  if (v->profiling) v->prof_launches += 1;
  return RF_OK;
}

int next_op(Batch& b) {
  if (b.n_ops >= b.max_ops) {
    std::fprintf(stderr, "refusion_b200: op record overflow (%d >= %d)\n", b.n_ops, b.max_ops);
    std::abort();
  }
  return b.n_ops++;
}

void flush_gc(Batch& b);

// A pending stream op runs on its own (k_stream) unless a footprint launch
// took it (op_fuse).
void flush_stream(Batch& b) {
  if (!b.st_pending) return;
  b.st_pending = false;
  rf_volume* v = b.v;
  ProfScope ps(v, 3);
  launch(k_stream, v->n_sms * 4, 256, 0, v->stream, v->T, b.st_p);
  if (v->profiling) v->prof_launches += 1;
}

void op_stream(Batch& b, const double c[3]) {
  rf_volume* v = b.v;
  const int gc = b.gc_pending;  // merged into this op's pass when it launches one
  b.gc_pending = -1;
  const int op = next_op(b);
  b.infos.push_back({0, -1});
  b.fparams.emplace_back();
  StreamParams p{};
  std::memcpy(p.old_c, b.center, sizeof(p.old_c));
  std::memcpy(p.new_c, c, sizeof(p.new_c));
  p.has_old = b.has_center;
  p.span = kBlockSide * v->cfg.voxel_size;
  p.radius2 = sqrt_le_bound(v->cfg.stream_radius);
  p.op_index = op;
  p.op = v->d_ops + op;
  p.ws = v->d_ws;
  // tiers are a function of the centre: an unchanged centre moves nothing
  const bool same = b.has_center && c[0] == b.center[0] && c[1] == b.center[1] && c[2] == b.center[2];
  // (a pending stream op of an unchanged centre stays mergeable: nothing
  // between them changes the blocks)
  if (!same) {
    flush_stream(b);
    if (gc >= 0) {
      ProfScope ps(v, 3);
      launch(k_gc_stream, v->n_sms * 4, 256, 0, v->stream, v->T, gc, &v->d_ops[gc].n_new,
             v->d_gc_stamp, v->gc_epoch, p);
      if (v->profiling) v->prof_launches += 1;
    } else {  // merged into the next footprint launch, or flushed
      b.st_pending = true;
      b.st_p = p;
    }
  } else if (gc >= 0) {
    b.gc_pending = gc;
    flush_gc(b);
  }
  // relocation (volume.py:358-364): centre moved more than one block span
  int reloc = 0;
  if (b.has_center) {
    const double dx = c[0] - b.center[0], dy = c[1] - b.center[1], dz = c[2] - b.center[2];
    const double moved = std::sqrt(dx * dx + dy * dy + dz * dz);
    if (moved > kBlockSide * v->cfg.voxel_size) reloc = 1;
  }
  b.streams.push_back({op, {c[0], c[1], c[2]}, reloc});
  b.has_center = true;
  std::memcpy(b.center, c, sizeof(b.center));
}

FootprintParams footprint_params(rf_volume* v, const Batch& b, const rf_kf_view* kf,
                                 const rf_pose* pose, int op) {
  FootprintParams p{};
  p.kf = to_view(kf);
  std::memcpy(p.R, pose->R, sizeof(p.R));
  std::memcpy(p.t, pose->t, sizeof(p.t));
  p.voxel_size = v->cfg.voxel_size;
  p.mu = v->cfg.mu;
  p.span = kBlockSide * v->cfg.voxel_size;
  p.inv_span = 1.0 / p.span;                       // volume.py:177
  p.min_z = 0.25 * v->cfg.voxel_size;              // volume.py:30, :170
  p.radius2 = sqrt_le_bound(v->cfg.stream_radius);
  std::memcpy(p.center, b.center, sizeof(p.center));
  p.has_center = b.has_center;
  p.n_steps = static_cast<int>(std::ceil(2.0 * v->cfg.mu / v->cfg.voxel_size)) + 1;  // :172
  p.shard_rank = v->cfg.shard_rank;
  p.shard_count = v->cfg.shard_count;
  p.epoch = ++v->epoch;
  if (v->epoch == 0xffffffffu) v->epoch = 1;  // stamps are reset lazily: 0 is "never"
  p.op_index = op;
  p.op = v->d_ops + op;
  p.ws = v->d_ws;
  return p;
}

void set_dim_bits(FuseParams& p) {
  const double w = static_cast<double>(p.kf.width), h = static_cast<double>(p.kf.height);
  std::memcpy(&p.w_bits, &w, sizeof(w));
  std::memcpy(&p.h_bits, &h, sizeof(h));
  // voxel-centre offsets (l + 0.5) * voxel_size (_kernels_cy.pyx:55-57)
  for (int l = 0; l < 8; ++l) p.hz[l] = (static_cast<double>(l) + 0.5) * p.voxel_size;
  // screened projection preconditions (rf_kernels.cuh, screen_coord)
  const double lim = 16384.0;
  p.fast_proj = p.kf.width < 16384 && p.kf.height < 16384 && std::fabs(p.kf.cx) < lim &&
                std::fabs(p.kf.cy) < lim;
}

FuseParams fuse_params(rf_volume* v, const rf_kf_view* kf, const rf_pose* pose, int op) {
  FuseParams p{};
  p.kf = to_view(kf);
  // rot_wc = pose.rotation.T (volume.py:260)
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) p.Rwc[3 * r + c] = pose->R[3 * c + r];
  std::memcpy(p.t, pose->t, sizeof(p.t));
  p.voxel_size = v->cfg.voxel_size;
  p.span = kBlockSide * v->cfg.voxel_size;
  p.mu = v->cfg.mu;
  p.eps_w = 1e-9;  // EPS_W, volume.py:26
  set_dim_bits(p);
  p.op_index = op;
  p.op = v->d_ops + op;
  p.ws = v->d_ws;
  p.shard_count = v->cfg.shard_count;
  return p;
}

int footprint_grid(rf_volume* v, const rf_kf_view* kf) {
  const long long tiles = static_cast<long long>((kf->width + kTile - 1) / kTile) *
                          ((kf->height + kTile - 1) / kTile);
  return static_cast<int>(std::max(1LL, std::min<long long>(tiles, v->fp_grid_cap)));
}

MemoKey memo_key(const rf_kf_view* kf, const rf_pose* pose) {
  MemoKey k;
  std::memset(&k, 0, sizeof(k));
  if (kf->memo_tag) {  // caller-supplied identity (planes uploaded per call)
    k.depth = reinterpret_cast<const void*>(static_cast<uintptr_t>(kf->memo_tag));
    k.weight = nullptr;
  } else {
    k.depth = kf->depth;
    k.weight = kf->weight;
  }
  k.width = kf->width;
  k.height = kf->height;
  k.intr[0] = kf->fx;
  k.intr[1] = kf->fy;
  k.intr[2] = kf->cx;
  k.intr[3] = kf->cy;
  std::memcpy(k.R, pose->R, sizeof(k.R));
  std::memcpy(k.t, pose->t, sizeof(k.t));
  return k;
}

void memo_evict_lru(rf_volume* v) {
  const MemoKey& old = v->memo_lru.back();
  auto it = v->memo.find(old);
  if (it != v->memo.end()) {
    v->memo_free.push_back(it->second.index);
    v->memo.erase(it);
  }
  v->memo_lru.pop_back();
}

void memo_release(rf_volume* v) {
  v->memo.clear();
  v->memo_lru.clear();
  v->memo_free.clear();
  if (v->memo_arena) {
    cudaStreamSynchronize(v->stream);  // kernels in flight may still read entries
    cudaFree(v->memo_arena);
  }
  v->memo_arena = nullptr;
  v->memo_slot_bytes = 0;
  v->memo_slot_cap = 0;
}

// Per-keyframe key capacity of a memo slot for npix-pixel keyframes (a
// sharded volume's entries hold the WHOLE footprint -- the contract is
// checked on every key -- recorded by its sampling pass, duplicates across
// pixel tiles included: room for one key per pixel).
int memo_cap_for(const rf_volume* v, long long npix) {
  return static_cast<int>(
      v->cfg.shard_count > 1 ? std::max(4096LL, npix)
                             : std::min<long long>(v->T.capacity, std::max(4096LL, npix / 3)));
}

// The memo arena, slots sized for `cap` keys each (allocated once).
bool memo_arena_alloc(rf_volume* v, int cap) {
  const size_t head = (sizeof(FpEntry) + 15) & ~size_t(15);
  const size_t slot = (head + sizeof(long long) * static_cast<size_t>(cap) + 255) & ~size_t(255);
  const size_t n = v->memo_budget / slot;
  if (n == 0) return false;
  if (cudaMalloc(&v->memo_arena, n * slot) != cudaSuccess) {
    cudaGetLastError();
    v->memo_arena = nullptr;
    v->memo_budget = 0;  // no memo on this device
    return false;
  }
  v->memo_slot_bytes = slot;
  v->memo_slot_cap = cap;
  v->memo_free.clear();
  for (size_t i = n; i-- > 0;) v->memo_free.push_back(static_cast<int>(i));
  return true;
}

// Returns the memo entry for (kf, pose) and whether it pre-existed.
FpEntry* memo_lookup(rf_volume* v, const rf_kf_view* kf, const rf_pose* pose, bool& existed) {
  existed = false;
  // (a sharded volume's entries hold the WHOLE footprint -- the contract is
  // checked on every key -- recorded by its sampling pass, duplicates
  // across pixel tiles included: room for one key per pixel)
  if (v->memo_budget == 0) return nullptr;
  const MemoKey key = memo_key(kf, pose);
  auto it = v->memo.find(key);
  if (it != v->memo.end()) {
    v->memo_lru.splice(v->memo_lru.begin(), v->memo_lru, it->second.lru);
    existed = true;
    return it->second.dev;
  }
  const int cap = memo_cap_for(v, static_cast<long long>(kf->width) * kf->height);
  if (!v->memo_arena && !memo_arena_alloc(v, cap)) return nullptr;  // first use
  if (cap > v->memo_slot_cap) return nullptr;
  if (v->memo_free.empty()) {
    if (v->memo_lru.empty()) return nullptr;
    memo_evict_lru(v);
  }
  const int index = v->memo_free.back();
  v->memo_free.pop_back();
  char* mem = v->memo_arena + static_cast<size_t>(index) * v->memo_slot_bytes;
  FpEntry* dev = reinterpret_cast<FpEntry*>(mem);
  // (its descriptor is initialised by the op's k_footprint: memo_fresh)
  v->memo_lru.push_front(key);
  MemoSlot ms;
  ms.dev = dev;
  ms.index = index;
  ms.lru = v->memo_lru.begin();
  v->memo.emplace(key, ms);
  return dev;
}


// A routed volume consumes exactly the footprints its last rf_route sent;
// the consumed inbox generation is emptied afterwards (on the stream, ahead
// of the next rf_route, which synchronises before the callers' barrier).
rf_status route_expect(rf_volume* v, int n) {
  if (!v->route_on || v->route_nops == n) return RF_OK;
  return fail(v, RF_INVALID_ARG,
              "routed volume: rf_route must send exactly this call's footprints first");
}

struct RouteConsume {
  rf_volume* v;
  ~RouteConsume() {
    if (!v->route_on) return;
    ProfScope ps(v, 3);
    launch(k_route_reset, 8, 256, 0, v->stream, v->route_own, v->route_lay,
           static_cast<int>(v->route_gen & 1));
    if (v->profiling) v->prof_launches += 1;
    v->route_nops = 0;
  }
};

// Launch the batched fuse kernel of mode kMode.
#if RF_KF_TMA
// Tensor map of one f64 keyframe plane [height][width] with the kTileW x
// kTileH box of the fuse kernels' keyframe tiles (cuTensorMapEncodeTiled
// through the runtime's driver entry point; no -lcuda).
bool plane_tensor_map(CUtensorMap* m, const double* base, int width, int height) {
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
            cudaSuccess || q != cudaDriverEntryPointSuccess || !f)
      return false;
    fn = reinterpret_cast<Encode>(f);
  }
  std::memset(m, 0, sizeof(*m));
  if (!base || (reinterpret_cast<uintptr_t>(base) & 15) || (width * 8) % 16 || width < kTileW ||
      height < kTileH)
    return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(width), static_cast<cuuint64_t>(height)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(width) * 8};
  const cuuint32_t box[2] = {kTileW, kTileH};
  const cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

constexpr size_t kFuseDynSmem = static_cast<size_t>(kFuseThreads / 32) * kTileWarpBytes + 128;
#endif

// Launch the batched fuse kernel of mode kMode.
template <int kMode>
void launch_fuse(rf_volume* v, const FuseParams& p) {
  if constexpr (kMode == kCheckRemove) {  // the de-integration check: its own lean kernel
    launch(k_check, v->check_grid, kFuseThreads, 0, v->stream, v->T, p);
  } else {
#if RF_KF_TMA
  CUtensorMap md, mw;
  FuseParams q = p;
  q.kf_tma = plane_tensor_map(&md, p.kf.depth, p.kf.width, p.kf.height) &&
             plane_tensor_map(&mw, p.kf.weight, p.kf.width, p.kf.height);
  launch(k_fuse<kMode>, v->fuse_grids[kMode], kFuseThreads, kFuseDynSmem, v->stream, v->T, q,
         md, mw);
#else
  launch(k_fuse<kMode>, v->fuse_grids[kMode], kFuseThreads, 0, v->stream, v->T, p);
#endif
  }
}

// Host keyframe planes (planes_on_host): copy each distinct keyframe of a
// call (one correction window, or one op) once, on the volume's copy stream,
// into a ring of device slots; the returned views carry device pointers and
// the slot's ready event (the compute stream waits on it just before that
// entry's first kernel).  A slot is refilled only after the compute stream
// passed its previous occupant's last consumer (stage_consumed, recorded by
// an earlier window).  Returns the slot per view (-1: device view).
constexpr int kStageSlots = 16;

// Room for `need` doubles in a staging slot (+ its events).  Growing
// synchronises the device (cudaFree): a connected shard reserves its slots
// up front (rf_reserve) so no call of the lockstep phase grows one while a
// peer waits in k_shard_sync.
template <typename Slot>
rf_status stage_slot_grow(rf_volume* v, Slot& sl, size_t need) {
  if (!v->copy_stream)
    RF_CUDA_TRY(v, cudaStreamCreateWithFlags(&v->copy_stream, cudaStreamNonBlocking));
  if (sl.cap < need) {
    RF_CUDA_TRY(v, cudaStreamSynchronize(v->copy_stream));
    RF_CUDA_TRY(v, cudaStreamSynchronize(v->stream));
    if (sl.buf) cudaFree(sl.buf);
    sl.buf = nullptr;
    RF_CUDA_TRY(v, cudaMalloc(&sl.buf, sizeof(double) * need));
    sl.cap = need;
  }
  if (!sl.ready) RF_CUDA_TRY(v, cudaEventCreateWithFlags(&sl.ready, cudaEventDisableTiming));
  if (!sl.consumed)
    RF_CUDA_TRY(v, cudaEventCreateWithFlags(&sl.consumed, cudaEventDisableTiming));
  if (!sl.color_ready)
    RF_CUDA_TRY(v, cudaEventCreateWithFlags(&sl.color_ready, cudaEventDisableTiming));
  return RF_OK;
}

rf_status stage_views(rf_volume* v, const rf_kf_view* in, int n, std::vector<rf_kf_view>& out,
                      std::vector<int>& slot_of) {
  out.assign(in, in + n);
  slot_of.assign(n, -1);
  v->upload_flag.clear();  // flags are looked up only for this call's staged views
  bool any = false;
  for (int i = 0; i < n; ++i) any |= in[i].planes_on_host != 0;
  if (!any) return RF_OK;
  if (!v->copy_stream)
    RF_CUDA_TRY(v, cudaStreamCreateWithFlags(&v->copy_stream, cudaStreamNonBlocking));
  // every entry of one call (window) must be resident at once
  const size_t ring = std::max<size_t>(kStageSlots, static_cast<size_t>(n));
  if (v->stage.size() < ring) v->stage.resize(ring);
  if (v->stage_flags_cap < v->stage.size()) {  // (all earlier work is complete here)
    RF_CUDA_TRY(v, cudaStreamSynchronize(v->copy_stream));
    if (v->d_stage_flags) cudaFree(v->d_stage_flags);
    v->d_stage_flags = nullptr;
    RF_CUDA_TRY(v, cudaMalloc(&v->d_stage_flags, sizeof(unsigned) * 2 * v->stage.size()));
    RF_CUDA_TRY(v, cudaMemset(v->d_stage_flags, 0, sizeof(unsigned) * 2 * v->stage.size()));
    v->stage_flags_cap = v->stage.size();
    for (auto& sl : v->stage) sl.gen = 0;
  }
  for (auto& sl : v->stage) sl.host = nullptr;
  for (int i = 0; i < n; ++i) {
    const rf_kf_view& k = in[i];
    if (!k.planes_on_host) continue;
    int reuse = -1;  // the same keyframe earlier in this batch
    for (int j = 0; j < i; ++j)
      if (slot_of[j] >= 0 && in[j].depth == k.depth && in[j].weight == k.weight &&
          in[j].color == k.color) {
        reuse = slot_of[j];
        break;
      }
    const size_t npix = static_cast<size_t>(k.width) * k.height;
    if (reuse < 0 || v->stage[reuse].host != k.depth) {
      const int s = v->stage_next;
      v->stage_next = (v->stage_next + 1) % static_cast<int>(v->stage.size());
      auto& sl = v->stage[s];
      const size_t need = npix * (k.color ? 5 : 2);
      {
        const rf_status gst = stage_slot_grow(v, sl, need);
        if (gst != RF_OK) return gst;
      }
      if (sl.used) cudaStreamWaitEvent(v->copy_stream, sl.consumed, 0);
      // depth + weight first: the footprint and the removal check need only
      // those, so they start while the colour plane is still in flight
      cudaMemcpyAsync(sl.buf, k.depth, sizeof(double) * npix, cudaMemcpyHostToDevice, v->copy_stream);
      cudaMemcpyAsync(sl.buf + npix, k.weight, sizeof(double) * npix, cudaMemcpyHostToDevice,
                      v->copy_stream);
      RF_CUDA_TRY(v, cudaEventRecord(sl.ready, v->copy_stream));
      sl.gen = sl.gen % 255 + 1;  // a byte value, never 0 (the flags' initial value)
      const unsigned val = sl.gen * 0x01010101u;
      unsigned* flag = v->d_stage_flags + 2 * s;
      cudaMemsetAsync(flag, static_cast<int>(sl.gen), sizeof(unsigned), v->copy_stream);
      v->upload_flag[sl.buf] = {flag, val};
      if (k.color) {
        cudaMemcpyAsync(sl.buf + 2 * npix, k.color, sizeof(double) * 3 * npix,
                        cudaMemcpyHostToDevice, v->copy_stream);
        RF_CUDA_TRY(v, cudaEventRecord(sl.color_ready, v->copy_stream));
        v->color_ready[sl.buf + 2 * npix] = sl.color_ready;
        cudaMemsetAsync(flag + 1, static_cast<int>(sl.gen), sizeof(unsigned), v->copy_stream);
        v->upload_flag[sl.buf + 2 * npix] = {flag + 1, val};
      }
      sl.used = true;
      sl.host = k.depth;
      reuse = s;
    }
    const auto& sl = v->stage[reuse];
    slot_of[i] = reuse;
    rf_kf_view& o = out[i];
    o.depth = sl.buf;
    o.weight = sl.buf + npix;
    o.color = k.color ? sl.buf + 2 * npix : nullptr;
    o.ready_event = sl.ready;
    o.planes_on_host = 0;
    // the host planes identify the keyframe for the footprint memo
    if (!o.memo_tag) o.memo_tag = reinterpret_cast<uintptr_t>(k.depth) * 0x9E3779B97F4A7C15ull ^
                                  reinterpret_cast<uintptr_t>(k.weight);
  }
  return RF_OK;
}

// The compute stream passed every use of view i's staged planes.
void stage_consumed(rf_volume* v, const std::vector<int>& slot_of, int i) {
  if (i < static_cast<int>(slot_of.size()) && slot_of[i] >= 0)
    cudaEventRecord(v->stage[slot_of[i]].consumed, v->stream);
}

// The upload flag of a staged plane, {nullptr, 0} for a caller-resident one.
std::pair<const unsigned*, unsigned> upload_flag_of(const rf_volume* v, const double* plane) {
  if (!plane || v->upload_flag.empty()) return {nullptr, 0u};
  auto it = v->upload_flag.find(plane);
  return it == v->upload_flag.end() ? std::pair<const unsigned*, unsigned>{nullptr, 0u}
                                    : it->second;
}

// A staged keyframe's colour plane may still be uploading: the kernels that
// read colour (integrate / removal apply) wait for it.
void wait_color(rf_volume* v, const rf_kf_view* kf) {
  if (!kf->color || v->color_ready.empty()) return;
  auto it = v->color_ready.find(kf->color);
  if (it != v->color_ready.end()) cudaStreamWaitEvent(v->stream, it->second, 0);
}

// mode: 0 integrate, 1 deintegrate, 2 allocate only.
void op_fuse(Batch& b, const rf_kf_view* kf, const rf_pose* pose, int mode, int entry) {
  rf_volume* v = b.v;
  flush_gc(b);
  // a pending stream op's scan rides on this op's footprint launch
  FpStream merged{};
  if (b.st_pending) {
    std::memcpy(merged.old_c, b.st_p.old_c, sizeof(merged.old_c));
    std::memcpy(merged.new_c, b.st_p.new_c, sizeof(merged.new_c));
    merged.has_old = b.st_p.has_old;
    merged.op = b.st_p.op;
    b.st_pending = false;
  }
  // staged planes: the op's first kernel waits on the upload flag on the
  // device; other events (a caller's own uploads) on the stream
  const auto up = upload_flag_of(v, kf->depth);
  const auto upc = upload_flag_of(v, kf->color);
  if (kf->ready_event && !up.first)
    cudaStreamWaitEvent(v->stream, static_cast<cudaEvent_t>(kf->ready_event), 0);
  const int op = next_op(b);
  b.infos.push_back({mode == 0 ? 1 : (mode == 1 ? 2 : 4), entry});
  FootprintParams fp = footprint_params(v, b, kf, pose, op);
  fp.st = merged;
  fp.wait_flag = up.first;
  fp.wait_val = up.second;
  bool existed = false;
  FpEntry* memo = nullptr;
  if (v->route_on) {  // the footprint arrives in this shard's inbox (k_route)
    const int idx = b.route_force >= 0 ? b.route_force : b.route_next++;
    const int par = static_cast<int>(v->route_gen & 1);
    const RouteLayout& L = v->route_lay;
    fp.route_keys = reinterpret_cast<const long long*>(v->route_own + L.keys_off(par, idx, 0));
    fp.route_counts = reinterpret_cast<const unsigned*>(v->route_own + L.count_off(par, idx, 0));
    fp.route_viol = reinterpret_cast<const long long*>(v->route_own + L.viol_off(par, idx));
    fp.route_segs = L.shards;
    fp.route_cap = L.cap;
  } else {
    memo = memo_lookup(v, kf, pose, existed);
    if (memo) {
      fp.memo_keys = reinterpret_cast<long long*>(reinterpret_cast<char*>(memo) +
                                                  ((sizeof(FpEntry) + 15) & ~size_t(15)));
      fp.memo_cap = v->memo_slot_cap;
      fp.memo_fresh = existed ? 0 : 1;
    }
  }
  int launches = 0;
  {
    ProfScope ps(v, 2);
    if (memo) {
      fp.kf_hash = &v->d_ops[op].kf_hash;
      fp.use_full = &v->d_ops[op].use_full;
      fp.memo = memo;
      if (existed) {  // the guard must be known before the cached keys are used
        const long long npix = static_cast<long long>(kf->width) * kf->height;
        launch(k_kf_hash, v->n_sms * 4, 256, 0, v->stream, kf->depth, kf->weight, npix,
               &v->d_ops[op].kf_hash, up.first, up.second);
        launches += 1;
      } else {  // a new entry samples the rays anyway: hash the planes there
        fp.hash_inline = 1;
      }
    }
    // cached key list or full ray sampling (decided on the device), then
    // the allocation of the missing blocks
    launch(k_footprint<false>, footprint_grid(v, kf), 256, 0, v->stream, v->T, fp);
    launch(k_commit, v->n_sms * 2, 256, 0, v->stream, v->T, fp);
    launches += 2;
  }
  FuseParams p = fuse_params(v, kf, pose, op);
  p.capture = memo;
  b.fparams.push_back(p);
  b.fparams.back().capture = nullptr;  // the fix-up relaunch must not re-capture
  if (v->profiling) v->prof_pixels += static_cast<long long>(kf->width) * kf->height;
  if (mode == 2) {
    p.alloc_only = 1;
    launch_fuse<kIntegrate>(v, p);
    if (v->profiling) v->prof_launches += launches + 1;
    return;
  }
  if (mode == 0) {
    if (upc.first) {  // the colour upload: waited for by the kernel
      p.wait_flag = upc.first;
      p.wait_val = upc.second;
    } else {
      wait_color(v, kf);
    }
    ProfScope ps(v, 0);
    launch_fuse<kIntegrate>(v, p);
    p.wait_flag = nullptr;
    launches += 1;
  } else {
    {
      ProfScope ps(v, 1);
      launch_fuse<kCheckRemove>(v, p);
    }
    p.capture = nullptr;
    launches += 1;
    if (v->sync_on) {  // the global verdict of this removal (every shard's check)
      SyncArgs sa{};
      for (int s = 0; s < v->cfg.shard_count; ++s) sa.peer[s] = v->sync_peer[s];
      sa.own = v->sync_own;
      sa.shards = v->cfg.shard_count;
      sa.parity = static_cast<int>(v->sync_gen & 1);
      sa.max_ops = v->sync_max_ops;
      ProfScope ps(v, 3);
      launch(k_shard_sync, 1, 32, 0, v->stream, sa, op, v->d_ops + op, v->d_ws,
             60ull * 2000000000ull);  // ~60 s at 2 GHz: a peer that never comes is an error
      launches += 1;
    }
    // the check read no colour; the removal does
    if (upc.first) {
      p.wait_flag = upc.first;
      p.wait_val = upc.second;
    } else {
      wait_color(v, kf);
    }
    {
      ProfScope ps(v, 4);
      launch_fuse<kApplyRemove>(v, p);
      launches += 1;
    }
  }
  if (v->profiling) v->prof_launches += launches;
}

// A GC op is launched lazily: merged with the stream op that follows it
// (k_gc_stream), or on its own before any other launch (flush_gc).
void flush_gc(Batch& b) {
  if (b.gc_pending < 0) return;
  flush_stream(b);  // a stream op before the GC counts the blocks the GC frees
  rf_volume* v = b.v;
  const int op = b.gc_pending;
  b.gc_pending = -1;
  // freed count lands in the op's n_new field
  ProfScope ps(v, 3);
  launch(k_gc, v->n_sms * 8, 256, 0, v->stream, v->T, op, v->d_ws, &v->d_ops[op].n_new,
         v->d_gc_stamp, v->gc_epoch);
  if (v->profiling) v->prof_launches += 1;
}

void op_gc(Batch& b) {
  rf_volume* v = b.v;
  flush_stream(b);
  flush_gc(b);
  const int op = next_op(b);
  b.infos.push_back({3, -1});
  b.fparams.emplace_back();
  b.gc_op = op;
  if (++v->gc_epoch == 0) {  // stamps wrapped: clear them
    cudaMemsetAsync(v->d_gc_stamp, 0, sizeof(unsigned) * v->cfg.hash_buckets, v->stream);
    v->gc_epoch = 1;
  }
  b.gc_pending = op;
}

// A connected shard's call that may de-integrate: a new sync generation;
// the previous call's parity is reset for the next call (all peers finished
// the previous call: the callers agree on every call's status).
rf_status sync_begin(rf_volume* v, int max_ops) {
  if (!v->sync_on) return RF_OK;
  if (max_ops > v->sync_max_ops)
    return fail(v, RF_INVALID_ARG, "shard sync: more ops in one call than the sync slots hold");
  ++v->sync_gen;
  launch(k_sync_reset, 8, 256, 0, v->stream, v->sync_own, v->sync_max_ops,
         static_cast<int>((v->sync_gen ^ 1u) & 1u));
  return RF_OK;
}

struct BatchOutcome {
  int err_kind = kErrNone;
  int err_op = -1;
};

// Synchronise once, read every op record, commit host streaming state for
// the ops that executed.
rf_status batch_end(Batch& b, BatchOutcome& out) {
  rf_volume* v = b.v;
  flush_stream(b);
  flush_gc(b);
  const int n = std::max(b.n_ops, 1);
  cudaMemcpyAsync(v->h_ops, v->d_ops, sizeof(OpCounters) * n, cudaMemcpyDeviceToHost, v->stream);
  cudaMemcpyAsync(v->h_ws, v->d_ws, sizeof(WinState), cudaMemcpyDeviceToHost, v->stream);
  RF_CUDA_TRY(v, cudaStreamSynchronize(v->stream));
  RF_CUDA_TRY(v, cudaGetLastError());
  out.err_kind = v->h_ws->err_kind;
  out.err_op = out.err_kind ? v->h_ws->err_op : -1;
  if (out.err_kind == kErrInconsistent) {
    // volume.py:331-333: blocks sorted before the failing one were removed
    // and re-added; the rest stays untouched.  The later ops were skipped,
    // so the failed op's touched list is still intact.
    launch_fuse<kRemoveReadd>(v, b.fparams[out.err_op]);
    RF_CUDA_TRY(v, cudaStreamSynchronize(v->stream));
    RF_CUDA_TRY(v, cudaGetLastError());
  }
  for (const PendingStream& s : b.streams) {
    if (out.err_kind && s.op > out.err_op) break;
    v->has_center = true;
    std::memcpy(v->center, s.c, sizeof(v->center));
    v->relocations += s.relocated;
  }
  if (v->profiling) {
    for (int i = 0; i < b.n_ops; ++i) {
      const int k = b.infos[i].kind;
      if (k == 2 && out.err_kind && i == out.err_op) v->prof_rem_ops += 1;  // it ran too
      if ((k == 1 || k == 2) && (!out.err_kind || i < out.err_op)) {
        const OpCounters& o = v->h_ops[i];
        v->prof_voxels += static_cast<long long>(o.voxels_updated);
        v->prof_blocks += static_cast<long long>(o.n_touched);
        const long long npix = static_cast<long long>(b.fparams[i].kf.width) *
                               b.fparams[i].kf.height;
        if (k == 1) {
          v->prof_int_vox += static_cast<long long>(o.voxels_updated);
          v->prof_int_pix += npix;
        } else {
          v->prof_rem_vox += static_cast<long long>(o.voxels_updated);
          v->prof_rem_pix += npix;
          v->prof_rem_ops += 1;
        }
      }
    }
  }
  return RF_OK;
}

rf_status status_of(rf_volume* v, int err_kind, const char* what) {
  switch (err_kind) {
    case kErrNone: return RF_OK;
    case kErrContract:
      return fail(v, RF_STREAMING_CONTRACT,
                  std::string(what) + ": a footprint block lies outside the active streaming "
                                      "sphere (host tier or beyond stream_radius), or stream() "
                                      "was never positioned");
    case kErrInconsistent:
      return fail(v, RF_INCONSISTENT,
                  std::string(what) + ": de-integration would drive a weight negative; the "
                                      "keyframe was not integrated with this pose");
    case kErrCapacity:
      return fail(v, RF_CAPACITY, std::string(what) + ": block pool capacity exhausted");
  }
  return fail(v, RF_CUDA, "unknown device error");
}

rf_status copy_new_keys(rf_volume* v, int op, int64_t* keys_host, int64_t cap) {
  const long long n = static_cast<long long>(v->h_ops[op].n_new);
  if (!keys_host || n == 0) return RF_OK;
  const long long m = std::min<long long>(n, cap);
  long long* d_keys = nullptr;
  RF_CUDA_TRY(v, cudaMallocAsync(&d_keys, sizeof(long long) * m + 8, v->stream));
  k_gather_keys<<<static_cast<int>((m + 255) / 256), 256, 0, v->stream>>>(v->T, v->T.new_list, m, d_keys);
  cudaMemcpyAsync(keys_host, d_keys, sizeof(long long) * m, cudaMemcpyDeviceToHost, v->stream);
  cudaFreeAsync(d_keys, v->stream);
  RF_CUDA_TRY(v, cudaStreamSynchronize(v->stream));
  return RF_OK;
}

}  // namespace

// ===========================================================================
// C ABI

extern "C" {

const char* rf_status_string(int status) {
  switch (status) {
    case RF_OK: return "ok";
    case RF_STREAMING_CONTRACT: return "streaming contract violated";
    case RF_INCONSISTENT: return "volume inconsistency";
    case RF_CAPACITY: return "block capacity exhausted";
    case RF_INVALID_ARG: return "invalid argument";
    case RF_CUDA: return "CUDA error";
  }
  return "unknown status";
}

const char* rf_last_error(const rf_volume* vol) { return vol ? vol->err.c_str() : ""; }

int64_t rf_block_hash(int64_t x, int64_t y, int64_t z, int64_t buckets) {
  if (buckets <= 0) return -1;
  return block_hash(x, y, z, buckets);
}

int32_t rf_key_owner(int64_t key, int32_t shard_count) {
  return shard_count <= 1 ? 0 : key_owner(key, shard_count);
}

rf_status rf_volume_create(const rf_config* cfg, rf_volume** out) {
  if (!cfg || !out) return RF_INVALID_ARG;
  *out = nullptr;
  if (!(cfg->voxel_size > 0.0) || !(cfg->mu >= 2.0 * cfg->voxel_size) ||
      !(cfg->stream_radius > cfg->mu) || cfg->hash_buckets <= 0 ||
      cfg->hash_buckets > 0x7fffffffLL || cfg->block_capacity <= 0 ||
      cfg->block_capacity > 0x3ffffff0LL || cfg->shard_count < 1 || cfg->shard_rank < 0 ||
      cfg->shard_rank >= cfg->shard_count)
    return RF_INVALID_ARG;
  rf_volume* v = new rf_volume();
  v->cfg = *cfg;
  if (cudaSetDevice(cfg->device) != cudaSuccess) {
    delete v;
    return RF_CUDA;
  }
  cudaDeviceGetAttribute(&v->n_sms, cudaDevAttrMultiProcessorCount, cfg->device);
  {  // the stream-ordered pool keeps what it has (memo entries, scratch): no
     // OS-level unmap / map between batches
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, cfg->device) == cudaSuccess) {
      unsigned long long thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  int occ[4] = {1, 1, 1, 1};
#if RF_KF_TMA
  const size_t dsm = kFuseDynSmem;
  cudaFuncSetAttribute(k_fuse<kIntegrate>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dsm));
  cudaFuncSetAttribute(k_fuse<kApplyRemove>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dsm));
  cudaFuncSetAttribute(k_fuse<kRemoveReadd>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dsm));
#else
  const size_t dsm = 0;
#endif
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[0], k_fuse<kIntegrate>, kFuseThreads, dsm);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[2], k_fuse<kApplyRemove>, kFuseThreads, dsm);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[3], k_fuse<kRemoveReadd>, kFuseThreads, dsm);
  for (int m = 0; m < 4; ++m) v->fuse_grids[m] = v->n_sms * std::max(occ[m], 1);
  {
    int oc = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oc, k_check, kFuseThreads, 0);
    v->check_grid = v->n_sms * std::max(oc, 1);
  }
  v->fuse_grid = v->fuse_grids[0];
  v->fp_grid_cap = v->n_sms * 8;
  const size_t cap = static_cast<size_t>(cfg->block_capacity);
  Table& T = v->T;
  T.buckets = cfg->hash_buckets;
  T.capacity = static_cast<int>(cap);
  T.pend_mask = kPendingSlots - 1;
  T.spill_cap = kSpillSlots;
  T.defer_cap = kDeferSlots;
  auto alloc = [&](void** p, size_t bytes) { return cudaMalloc(p, bytes) == cudaSuccess; };
  bool ok = alloc(reinterpret_cast<void**>(&T.heads), sizeof(int) * cfg->hash_buckets) &&
            alloc(reinterpret_cast<void**>(&T.keys), sizeof(long long) * cap) &&
            alloc(reinterpret_cast<void**>(&T.next), sizeof(int) * cap) &&
            alloc(reinterpret_cast<void**>(&T.nz), sizeof(int) * cap) &&
            alloc(reinterpret_cast<void**>(&T.stamp), sizeof(unsigned) * cap) &&
            alloc(reinterpret_cast<void**>(&T.free_stack), sizeof(int) * cap) &&
            alloc(reinterpret_cast<void**>(&T.returned), sizeof(int) * cap) &&
            alloc(reinterpret_cast<void**>(&T.touched), sizeof(int) * cap) &&
            alloc(reinterpret_cast<void**>(&T.touched_keys), sizeof(long long) * cap) &&
            alloc(reinterpret_cast<void**>(&T.tpos), sizeof(int) * cap) &&
            alloc(reinterpret_cast<void**>(&T.new_list), sizeof(int) * cap) &&
            alloc(reinterpret_cast<void**>(&T.pend_tab), sizeof(long long) * kPendingSlots) &&
            alloc(reinterpret_cast<void**>(&T.pend_keys), sizeof(long long) * kPendingSlots) &&
            alloc(reinterpret_cast<void**>(&T.pend_idx), sizeof(int) * kPendingSlots) &&
            alloc(reinterpret_cast<void**>(&T.spill_keys), sizeof(long long) * kSpillSlots) &&
            alloc(reinterpret_cast<void**>(&T.defer), sizeof(unsigned long long) * kDeferSlots) &&
            alloc(reinterpret_cast<void**>(&T.alloc), sizeof(AllocState)) &&
            alloc(reinterpret_cast<void**>(&T.pool), sizeof(double) * kBlockDoubles * cap) &&
            alloc(reinterpret_cast<void**>(&v->d_ws), sizeof(WinState)) &&
            alloc(reinterpret_cast<void**>(&v->d_gc_stamp), sizeof(unsigned) * cfg->hash_buckets) &&
            alloc(reinterpret_cast<void**>(&v->d_u64), sizeof(unsigned long long) * 8) &&
            alloc(reinterpret_cast<void**>(&v->d_f64), sizeof(double) * 8) &&
            cudaMallocHost(&v->h_ws, sizeof(WinState)) == cudaSuccess &&
            cudaMallocHost(&v->h_u64, sizeof(unsigned long long) * 8) == cudaSuccess &&
            cudaMallocHost(&v->h_f64, sizeof(double) * 8) == cudaSuccess &&
            cudaMallocHost(&v->h_alloc, sizeof(AllocState)) == cudaSuccess;
  if (!ok) {
    rf_volume_destroy(v);
    return RF_CAPACITY;
  }
  cudaMemset(T.heads, 0xff, sizeof(int) * cfg->hash_buckets);
  cudaMemset(T.keys, 0xff, sizeof(long long) * cap);
  cudaMemset(T.pend_tab, 0xff, sizeof(long long) * kPendingSlots);
  cudaMemset(T.nz, 0, sizeof(int) * cap);
  cudaMemset(v->d_gc_stamp, 0, sizeof(unsigned) * cfg->hash_buckets);
  cudaMemset(T.stamp, 0, sizeof(unsigned) * cap);
  cudaMemset(T.alloc, 0, sizeof(AllocState));
  cudaMemset(v->d_ws, 0, sizeof(WinState));
  if (ensure_ops(v, 64) != RF_OK || cudaDeviceSynchronize() != cudaSuccess) {
    rf_volume_destroy(v);
    return RF_CUDA;
  }
  *out = v;
  return RF_OK;
}

rf_status rf_volume_destroy(rf_volume* v) {
  if (!v) return RF_OK;
  cudaSetDevice(v->cfg.device);
  // this volume's own work only (other volumes' kernels may be waiting for
  // their peers inside k_shard_sync)
  cudaStreamSynchronize(v->stream);
  if (v->copy_stream) cudaStreamSynchronize(v->copy_stream);
  Table& T = v->T;
  void* ptrs[] = {T.heads, T.keys, T.next, T.nz, T.stamp, T.free_stack, T.returned, T.touched, T.touched_keys, T.tpos,
                  T.new_list, T.pend_tab, T.pend_keys, T.pend_idx, T.spill_keys, T.defer, T.alloc, T.pool, v->d_ws, v->d_u64, v->d_f64, v->d_ops, v->d_wsums, v->d_gc_stamp};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  void* hptrs[] = {v->h_ws, v->h_u64, v->h_f64, v->h_alloc, v->h_ops};
  for (void* p : hptrs)
    if (p) cudaFreeHost(p);
  for (auto& e : v->events) {
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  for (auto e : v->event_pool) cudaEventDestroy(e);
  memo_release(v);
  for (auto& sl : v->stage) {
    if (sl.buf) cudaFree(sl.buf);
    if (sl.ready) cudaEventDestroy(sl.ready);
    if (sl.color_ready) cudaEventDestroy(sl.color_ready);
    if (sl.consumed) cudaEventDestroy(sl.consumed);
  }
  if (v->copy_stream) cudaStreamDestroy(v->copy_stream);
  if (v->d_stage_flags) cudaFree(v->d_stage_flags);
  for (int s = 0; s < kMaxShards; ++s) {
    if (v->route_ipc[s]) cudaIpcCloseMemHandle(v->route_peer[s]);
    if (v->sync_ipc[s]) cudaIpcCloseMemHandle(v->sync_peer[s]);
    for (int a = 0; a < 4; ++a)
      if (v->mesh_ipc[s][a]) cudaIpcCloseMemHandle(v->mesh_ipc[s][a]);
  }
  if (v->route_own) cudaFree(v->route_own);
  if (v->sync_own) cudaFree(v->sync_own);
  delete v;
  return RF_OK;
}

rf_status rf_set_cuda_stream(rf_volume* v, void* stream) {
  if (!v) return RF_INVALID_ARG;
  v->stream = static_cast<cudaStream_t>(stream);
  return RF_OK;
}

rf_status rf_stream(rf_volume* v, const double center[3], rf_stream_result* result) {
  if (!v || !center) return RF_INVALID_ARG;
  cudaSetDevice(v->cfg.device);
  Batch b;
  rf_status st = batch_begin(v, b, 1);
  if (st != RF_OK) return st;
  op_stream(b, center);
  BatchOutcome o;
  st = batch_end(b, o);
  if (st != RF_OK) return st;
  if (result) {
    result->streamed_in = static_cast<int64_t>(v->h_ops[0].streamed_in);
    result->streamed_out = static_cast<int64_t>(v->h_ops[0].streamed_out);
    result->relocated = b.streams[0].relocated;
  }
  return RF_OK;
}

rf_status rf_footprint(rf_volume* v, const rf_kf_view* kf, const rf_pose* pose, int64_t* keys_host,
                       int64_t cap, int64_t* n_out) {
  if (!v || !valid_kf(kf) || !pose || !n_out) return RF_INVALID_ARG;
  cudaSetDevice(v->cfg.device);
  std::vector<rf_kf_view> staged;
  std::vector<int> slot_of;
  {
    const rf_status sst = stage_views(v, kf, 1, staged, slot_of);
    if (sst != RF_OK) return sst;
    kf = staged.data();
  }
  Batch b;
  rf_status st = batch_begin(v, b, 1);
  if (st != RF_OK) return st;
  const long long npix = static_cast<long long>(kf->width) * kf->height;
  if (kf->ready_event) cudaStreamWaitEvent(v->stream, static_cast<cudaEvent_t>(kf->ready_event), 0);
  FootprintParams p = footprint_params(v, b, kf, pose, 0);
  long long dcap = npix * 4 + 1024;
  for (int attempt = 0; attempt < 2; ++attempt) {
    long long* d_keys = nullptr;
    RF_CUDA_TRY(v, cudaMallocAsync(&d_keys, sizeof(long long) * dcap, v->stream));
    cudaMemsetAsync(v->d_u64, 0, sizeof(unsigned long long), v->stream);
    p.dry_keys = d_keys;
    p.dry_count = v->d_u64;
    p.dry_cap = dcap;
    k_footprint<true><<<footprint_grid(v, kf), 256, 0, v->stream>>>(v->T, p);
    cudaMemcpyAsync(v->h_u64, v->d_u64, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                    v->stream);
    RF_CUDA_TRY(v, cudaStreamSynchronize(v->stream));
    const long long got = static_cast<long long>(v->h_u64[0]);
    if (got <= dcap) {
      std::vector<long long> keys(static_cast<size_t>(got));
      if (got)
        cudaMemcpyAsync(keys.data(), d_keys, sizeof(long long) * got, cudaMemcpyDeviceToHost,
                        v->stream);
      cudaFreeAsync(d_keys, v->stream);
      RF_CUDA_TRY(v, cudaStreamSynchronize(v->stream));
      std::sort(keys.begin(), keys.end());  // np.unique, volume.py:191-193
      keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
      *n_out = static_cast<int64_t>(keys.size());
      if (keys_host)
        std::memcpy(keys_host, keys.data(),
                    sizeof(long long) * std::min<long long>(cap, static_cast<long long>(keys.size())));
      return RF_OK;
    }
    cudaFreeAsync(d_keys, v->stream);
    dcap = got + 1024;
  }
  return fail(v, RF_CUDA, "footprint scratch sizing failed");
}


// ---- routed footprints (hash-sharded volumes, k_route) --------------------

rf_status rf_route_setup(rf_volume* v, int32_t max_ops, int64_t cap_keys, void** inbox,
                         uint64_t* bytes) {
  if (!v || max_ops <= 0 || cap_keys <= 0 || cap_keys > (1LL << 30) || v->cfg.shard_count < 2 ||
      v->cfg.shard_count > kMaxShards)
    return RF_INVALID_ARG;
  cudaSetDevice(v->cfg.device);
  if (v->route_own) return fail(v, RF_INVALID_ARG, "rf_route_setup: inbox already set up");
  RouteLayout L{max_ops, v->cfg.shard_count, static_cast<int>(cap_keys)};
  void* mem = nullptr;
  RF_CUDA_TRY(v, cudaMalloc(&mem, L.bytes()));
  v->route_own = static_cast<char*>(mem);
  v->route_lay = L;
  for (int par = 0; par < 2; ++par)
    k_route_reset<<<8, 256, 0, v->stream>>>(v->route_own, L, par);
  RF_CUDA_TRY(v, cudaStreamSynchronize(v->stream));
  if (inbox) *inbox = mem;
  if (bytes) *bytes = L.bytes();
  return RF_OK;
}

rf_status rf_route_connect(rf_volume* v, void* const* inboxes) {
  if (!v || !inboxes || !v->route_own) return RF_INVALID_ARG;
  if (inboxes[v->cfg.shard_rank] != v->route_own)
    return fail(v, RF_INVALID_ARG, "rf_route_connect: own inbox mismatch");
  for (int s = 0; s < v->cfg.shard_count; ++s) {
    if (!inboxes[s]) return RF_INVALID_ARG;
    v->route_peer[s] = static_cast<char*>(inboxes[s]);
  }
  v->route_on = true;
  return RF_OK;
}

rf_status rf_route_ipc_handle(rf_volume* v, void* handle) {
  if (!v || !handle || !v->route_own) return RF_INVALID_ARG;
  cudaSetDevice(v->cfg.device);
  cudaIpcMemHandle_t h;
  RF_CUDA_TRY(v, cudaIpcGetMemHandle(&h, v->route_own));
  std::memcpy(handle, &h, sizeof(h));
  return RF_OK;
}

rf_status rf_route_ipc_open(rf_volume* v, const void* handles) {
  if (!v || !handles || !v->route_own) return RF_INVALID_ARG;
  cudaSetDevice(v->cfg.device);
  const int G = v->cfg.shard_count;
  std::vector<void*> ptrs(G, nullptr);
  for (int s = 0; s < G; ++s) {
    if (s == v->cfg.shard_rank) {
      ptrs[s] = v->route_own;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const char*>(handles) + s * sizeof(h), sizeof(h));
    RF_CUDA_TRY(v, cudaIpcOpenMemHandle(&ptrs[s], h, cudaIpcMemLazyEnablePeerAccess));
    v->route_ipc[s] = true;
  }
  return rf_route_connect(v, ptrs.data());
}

rf_status rf_route(rf_volume* v, int32_t n, const rf_kf_view* kfs, const rf_pose* poses,
                   const double* centers) {
  if (!v || n < 0 || (n > 0 && (!kfs || !poses))) return RF_INVALID_ARG;
  if (!v->route_on) return fail(v, RF_INVALID_ARG, "rf_route: inbox not connected");
  if (n > v->route_lay.max_ops) return fail(v, RF_INVALID_ARG, "rf_route: more ops than the inbox holds");
  for (int i = 0; i < n; ++i)
    if (!valid_kf(&kfs[i])) return RF_INVALID_ARG;
  cudaSetDevice(v->cfg.device);
  std::vector<rf_kf_view> staged;
  std::vector<int> slot_of;
  {
    const rf_status sst = stage_views(v, kfs, n, staged, slot_of);
    if (sst != RF_OK) return sst;
  }
  ++v->route_gen;
  RouteArgs r{};
  for (int s = 0; s < v->cfg.shard_count; ++s) r.peer[s] = v->route_peer[s];
  r.lay = v->route_lay;
  r.parity = static_cast<int>(v->route_gen & 1);
  r.rank = v->cfg.shard_rank;
  for (int i = 0; i < n; ++i) {
    const rf_kf_view* kf = &staged[i];
    if (kf->ready_event) cudaStreamWaitEvent(v->stream, static_cast<cudaEvent_t>(kf->ready_event), 0);
    Batch b;  // only the centre is read
    b.has_center = centers ? true : v->has_center;
    std::memcpy(b.center, centers ? centers + 3 * i : v->center, sizeof(b.center));
    FootprintParams fp = footprint_params(v, b, kf, &poses[i], 0);
    fp.op = nullptr;
    fp.ws = nullptr;
    r.op = i;
    const long long tiles = static_cast<long long>((kf->width + kTile - 1) / kTile) *
                            ((kf->height + kTile - 1) / kTile);
    const long long mine = (tiles + v->cfg.shard_count - 1) / v->cfg.shard_count;
    // enough CTAs to fill the GPU (8 per SM): split each tile by step range
    r.parts = static_cast<int>(std::max(1LL, std::min<long long>(
        std::min(8, fp.n_steps), v->fp_grid_cap / std::max(1LL, mine))));
    const int grid = static_cast<int>(
        std::max(1LL, std::min<long long>(mine * r.parts, v->fp_grid_cap)));
    ProfScope ps(v, 2);
    launch(k_route, grid, 256, 0, v->stream, fp, r);
    if (v->profiling) v->prof_launches += 1;
  }
  RF_CUDA_TRY(v, cudaStreamSynchronize(v->stream));  // peers read after the callers' barrier
  v->route_nops = n;
  return RF_OK;
}

// ---- cross-shard removal verdicts (k_shard_sync) ---------------------------

rf_status rf_shard_sync_setup(rf_volume* v, int32_t max_ops, void** slots, uint64_t* bytes) {
  if (!v || max_ops <= 0 || v->cfg.shard_count < 2 || v->cfg.shard_count > kMaxShards)
    return RF_INVALID_ARG;
  cudaSetDevice(v->cfg.device);
  if (v->sync_own) return fail(v, RF_INVALID_ARG, "rf_shard_sync_setup: already set up");
  const size_t n = 2 * static_cast<size_t>(max_ops) * sizeof(SyncSlot);
  void* mem = nullptr;
  RF_CUDA_TRY(v, cudaMalloc(&mem, n));
  v->sync_own = static_cast<SyncSlot*>(mem);
  v->sync_max_ops = max_ops;
  for (int par = 0; par < 2; ++par)
    k_sync_reset<<<8, 256, 0, v->stream>>>(v->sync_own, max_ops, par);
  RF_CUDA_TRY(v, cudaStreamSynchronize(v->stream));
  if (slots) *slots = mem;
  if (bytes) *bytes = n;
  return RF_OK;
}

rf_status rf_shard_sync_connect(rf_volume* v, void* const* slots) {
  if (!v || !slots || !v->sync_own) return RF_INVALID_ARG;
  if (slots[v->cfg.shard_rank] != v->sync_own)
    return fail(v, RF_INVALID_ARG, "rf_shard_sync_connect: own slots mismatch");
  for (int s = 0; s < v->cfg.shard_count; ++s) {
    if (!slots[s]) return RF_INVALID_ARG;
    v->sync_peer[s] = static_cast<SyncSlot*>(slots[s]);
  }
  v->sync_on = true;
  return RF_OK;
}

rf_status rf_shard_sync_ipc_handle(rf_volume* v, void* handle) {
  if (!v || !handle || !v->sync_own) return RF_INVALID_ARG;
  cudaSetDevice(v->cfg.device);
  cudaIpcMemHandle_t h;
  RF_CUDA_TRY(v, cudaIpcGetMemHandle(&h, v->sync_own));
  std::memcpy(handle, &h, sizeof(h));
  return RF_OK;
}

rf_status rf_shard_sync_ipc_open(rf_volume* v, const void* handles) {
  if (!v || !handles || !v->sync_own) return RF_INVALID_ARG;
  cudaSetDevice(v->cfg.device);
  const int G = v->cfg.shard_count;
  std::vector<void*> ptrs(G, nullptr);
  for (int s = 0; s < G; ++s) {
    if (s == v->cfg.shard_rank) {
      ptrs[s] = v->sync_own;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const char*>(handles) + s * sizeof(h), sizeof(h));
    RF_CUDA_TRY(v, cudaIpcOpenMemHandle(&ptrs[s], h, cudaIpcMemLazyEnablePeerAccess));
    v->sync_ipc[s] = true;
  }
  return rf_shard_sync_connect(v, ptrs.data());
}

rf_status rf_reserve(rf_volume* v, int32_t width, int32_t height, int32_t max_ops) {
  if (!v || width <= 0 || height <= 0 || max_ops <= 0 || max_ops > kMaxWindowOps * 8 ||
      static_cast<long long>(width) * height >= (1LL << 31))
    return RF_INVALID_ARG;
  cudaSetDevice(v->cfg.device);
  rf_status st = ensure_ops(v, max_ops);
  if (st != RF_OK) return st;
  const long long npix = static_cast<long long>(width) * height;
  if (v->stage.size() < static_cast<size_t>(kStageSlots)) v->stage.resize(kStageSlots);
  for (auto& sl : v->stage) {
    st = stage_slot_grow(v, sl, static_cast<size_t>(npix) * 5);
    if (st != RF_OK) return st;
  }
  if (v->memo_budget > 0 && !v->memo_arena) memo_arena_alloc(v, memo_cap_for(v, npix));
  RF_CUDA_TRY(v, cudaDeviceSynchronize());
  return RF_OK;
}

rf_status rf_allocate(rf_volume* v, const rf_kf_view* kf, const rf_pose* pose,
                      int64_t* new_keys_host, int64_t cap, int64_t* n_new) {
  if (!v || !valid_kf(kf) || !pose) return RF_INVALID_ARG;
  cudaSetDevice(v->cfg.device);
  std::vector<rf_kf_view> staged;
  std::vector<int> slot_of;
  {
    const rf_status sst = stage_views(v, kf, 1, staged, slot_of);
    if (sst != RF_OK) return sst;
    kf = staged.data();
  }
  if (route_expect(v, 1) != RF_OK) return RF_INVALID_ARG;
  RouteConsume rc{v};
  Batch b;
  rf_status st = batch_begin(v, b, 1);
  if (st != RF_OK) return st;
  op_fuse(b, kf, pose, 2, 0);
  BatchOutcome o;
  st = batch_end(b, o);
  if (st != RF_OK) return st;
  if (o.err_kind) return status_of(v, o.err_kind, "allocate_blocks");
  if (n_new) *n_new = static_cast<int64_t>(v->h_ops[0].n_new);
  return copy_new_keys(v, 0, new_keys_host, cap);
}

rf_status rf_integrate(rf_volume* v, const rf_kf_view* kf, const rf_pose* pose,
                       rf_op_result* result, int64_t* new_keys_host, int64_t new_cap) {
  if (!v || !valid_kf(kf) || !pose) return RF_INVALID_ARG;
  cudaSetDevice(v->cfg.device);
  std::vector<rf_kf_view> staged;
  std::vector<int> slot_of;
  {
    const rf_status sst = stage_views(v, kf, 1, staged, slot_of);
    if (sst != RF_OK) return sst;
    kf = staged.data();
  }
  if (route_expect(v, 1) != RF_OK) return RF_INVALID_ARG;
  RouteConsume rc{v};
  Batch b;
  rf_status st = batch_begin(v, b, 1);
  if (st != RF_OK) return st;
  op_fuse(b, kf, pose, 0, 0);
  BatchOutcome o;
  st = batch_end(b, o);
  if (st != RF_OK) return st;
  if (o.err_kind) return status_of(v, o.err_kind, "integrate");
  if (result) {
    result->blocks_touched = static_cast<int64_t>(v->h_ops[0].n_touched);
    result->voxels_updated = static_cast<int64_t>(v->h_ops[0].voxels_updated);
    result->n_new = static_cast<int64_t>(v->h_ops[0].n_new);
  }
  return copy_new_keys(v, 0, new_keys_host, new_cap);
}

rf_status rf_deintegrate(rf_volume* v, const rf_kf_view* kf, const rf_pose* pose,
                         rf_op_result* result) {
  if (!v || !valid_kf(kf) || !pose) return RF_INVALID_ARG;
  cudaSetDevice(v->cfg.device);
  std::vector<rf_kf_view> staged;
  std::vector<int> slot_of;
  {
    const rf_status sst = stage_views(v, kf, 1, staged, slot_of);
    if (sst != RF_OK) return sst;
    kf = staged.data();
  }
  if (route_expect(v, 1) != RF_OK) return RF_INVALID_ARG;
  RouteConsume rc{v};
  Batch b;
  rf_status st = batch_begin(v, b, 1);
  if (st != RF_OK) return st;
  st = sync_begin(v, 1);
  if (st != RF_OK) return st;
  op_fuse(b, kf, pose, 1, 0);
  BatchOutcome o;
  st = batch_end(b, o);
  if (st != RF_OK) return st;
  if (result) {
    result->blocks_touched = static_cast<int64_t>(v->h_ops[0].n_touched);
    result->voxels_updated = static_cast<int64_t>(v->h_ops[0].voxels_updated);
    result->n_new = static_cast<int64_t>(v->h_ops[0].n_new);
  }
  return status_of(v, o.err_kind, "deintegrate");
}

rf_status rf_correct_windows(rf_volume* v, int32_t n_windows, const int32_t* sizes,
                             const rf_kf_view* kfs, const rf_pose* old_poses,
                             const rf_pose* new_poses, const double* next_center,
                             rf_window_result* result) {
  if (!v || n_windows < 0 || (n_windows > 0 && !sizes)) return RF_INVALID_ARG;
  long long total = 0;
  for (int w = 0; w < n_windows; ++w) {
    if (sizes[w] < 0) return RF_INVALID_ARG;
    total += sizes[w];
  }
  if (total > kMaxWindowOps || n_windows > kMaxWindowOps)
    return fail(v, RF_INVALID_ARG, "too many entries in one call");
  if (total > 0 && (!kfs || !old_poses || !new_poses)) return RF_INVALID_ARG;
  for (long long i = 0; i < total; ++i)
    if (!valid_kf(&kfs[i])) return RF_INVALID_ARG;
  cudaSetDevice(v->cfg.device);
  rf_window_result r{};
  r.failed_entry = -1;
  r.failed_phase = -1;
  r.failed_window = -1;
  // routed: per window, its m removal footprints then its m integration ones
  if (route_expect(v, static_cast<int>(2 * total)) != RF_OK) return RF_INVALID_ARG;
  RouteConsume rc{v};
  Batch b;
  // per window: stream(old0) + m x (stream, deint) + stream(new0) + m x (stream, int) + gc
  rf_status st = batch_begin(v, b, static_cast<int>(4 * total + 3 * n_windows + 1));
  if (st != RF_OK) return st;
  st = sync_begin(v, static_cast<int>(4 * total + 3 * n_windows + 1));
  if (st != RF_OK) return st;
  // each window is reintegration._correct_entries (reintegration.py:156-181)
  long long base = 0;
  for (int w = 0; w < n_windows; ++w) {
    const int m = sizes[w];
    if (m == 0) continue;  // :161-162
    // host planes: staged per window (uploads overlap earlier windows' work)
    std::vector<rf_kf_view> staged;
    std::vector<int> slot_of;
    {
      const rf_status sst = stage_views(v, kfs + base, m, staged, slot_of);
      if (sst != RF_OK) return sst;
    }
    const rf_kf_view* k = staged.data();
    const rf_pose* o = old_poses + base;
    const rf_pose* n = new_poses + base;
    op_stream(b, o[0].t);
    for (int i = 0; i < m; ++i) {
      op_stream(b, o[i].t);
      op_fuse(b, &k[i], &o[i], 1, i);
      b.infos.back().window = w;
    }
    op_stream(b, n[0].t);
    for (int i = 0; i < m; ++i) {
      op_stream(b, n[i].t);
      op_fuse(b, &k[i], &n[i], 0, i);
      b.infos.back().window = w;
      stage_consumed(v, slot_of, i);  // last use of its planes
    }
    op_gc(b);
    b.infos.back().window = w;
    base += m;
  }
  if (next_center) op_stream(b, next_center);  // correct_window / correct_topk
  BatchOutcome out;
  st = batch_end(b, out);
  if (st != RF_OK) return st;
  for (int i = 0; i < b.n_ops; ++i) {
    if (out.err_kind && i > out.err_op) break;
    const OpInfo& inf = b.infos[i];
    if (inf.kind == 1 || inf.kind == 2) {
      r.blocks_touched += static_cast<int64_t>(v->h_ops[i].n_touched);
      r.n_new += static_cast<int64_t>(v->h_ops[i].n_new);
      if (inf.kind == 1) r.voxels_updated += static_cast<int64_t>(v->h_ops[i].voxels_updated);
    } else if (inf.kind == 3) {
      r.gc_freed += static_cast<int64_t>(v->h_ops[i].n_new);
    }
  }
  if (!out.err_kind) {
    r.status = RF_OK;
    r.n_corrected = total;
    if (result) *result = r;
    return RF_OK;
  }
  const OpInfo& bad = b.infos[out.err_op];
  r.failed_entry = bad.entry;
  r.failed_phase = bad.kind == 2 ? 0 : 1;
  r.failed_window = bad.window;
  long long wbase = 0;
  for (int w = 0; w < bad.window; ++w) {
    wbase += sizes[w];
    r.n_corrected += sizes[w];
  }
  rf_status wst = status_of(v, out.err_kind, bad.kind == 2 ? "deintegrate" : "integrate");
  if (out.err_kind == kErrInconsistent && bad.kind == 2 && bad.entry > 0) {
    // reintegration.py:170-174: re-integrate what was already removed
    const std::string msg = v->err;
    std::vector<rf_kf_view> staged;
    std::vector<int> slot_of;
    st = stage_views(v, kfs + wbase, bad.entry, staged, slot_of);
    if (st != RF_OK) return st;
    Batch rb;
    st = batch_begin(v, rb, 2 * bad.entry);
    if (st != RF_OK) return st;
    for (int i = 0; i < bad.entry; ++i) {
      op_stream(rb, old_poses[wbase + i].t);
      rb.route_force = static_cast<int>(2 * wbase + i);  // routed: the removal's footprint
      op_fuse(rb, &staged[i], &old_poses[wbase + i], 0, i);
    }
    BatchOutcome ro;
    st = batch_end(rb, ro);
    if (st != RF_OK) return st;
    if (ro.err_kind) {
      wst = status_of(v, ro.err_kind, "integrate (rollback)");
    } else {
      v->err = msg;
    }
  }
  r.status = wst;
  if (result) *result = r;
  return wst;
}

rf_status rf_correct(rf_volume* v, int32_t m, const rf_kf_view* kfs, const rf_pose* old_poses,
                     const rf_pose* new_poses, const double* next_center,
                     rf_window_result* result) {
  if (m < 0) return RF_INVALID_ARG;
  return rf_correct_windows(v, 1, &m, kfs, old_poses, new_poses, next_center, result);
}

rf_status rf_garbage_collect(rf_volume* v, int64_t* freed) {
  if (!v) return RF_INVALID_ARG;
  cudaSetDevice(v->cfg.device);
  Batch b;
  rf_status st = batch_begin(v, b, 1);
  if (st != RF_OK) return st;
  op_gc(b);
  BatchOutcome o;
  st = batch_end(b, o);
  if (st != RF_OK) return st;
  if (freed) *freed = static_cast<int64_t>(v->h_ops[0].n_new);
  return RF_OK;
}

rf_status rf_total_weight(rf_volume* v, double* out) {
  if (!v || !out) return RF_INVALID_ARG;
  cudaSetDevice(v->cfg.device);
  if (!v->d_wsums) RF_CUDA_TRY(v, cudaMalloc(&v->d_wsums, sizeof(double) * v->T.capacity));
  k_wsum_blocks<<<v->n_sms * 8, 256, 0, v->stream>>>(v->T, v->d_wsums);
  k_ordered_sum<<<1, 256, 0, v->stream>>>(v->T, v->d_wsums, v->d_f64);
  cudaMemcpyAsync(v->h_f64, v->d_f64, sizeof(double), cudaMemcpyDeviceToHost, v->stream);
  RF_CUDA_TRY(v, cudaStreamSynchronize(v->stream));
  *out = v->h_f64[0];
  return RF_OK;
}

rf_status rf_counters_get(rf_volume* v, rf_counters* out) {
  if (!v || !out) return RF_INVALID_ARG;
  cudaSetDevice(v->cfg.device);
  cudaMemsetAsync(v->d_u64, 0, sizeof(unsigned long long), v->stream);
  if (v->has_center)
    k_count_active<<<v->n_sms * 4, 256, 0, v->stream>>>(v->T, v->center[0], v->center[1],
                                                        v->center[2],
                                                        kBlockSide * v->cfg.voxel_size,
                                                        sqrt_le_bound(v->cfg.stream_radius),
                                                        v->d_u64);
  cudaMemcpyAsync(v->h_alloc, v->T.alloc, sizeof(AllocState), cudaMemcpyDeviceToHost, v->stream);
  cudaMemcpyAsync(v->h_u64, v->d_u64, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                  v->stream);
  RF_CUDA_TRY(v, cudaStreamSynchronize(v->stream));
  out->blocks_streamed_in = static_cast<int64_t>(v->h_alloc->total_streamed_in);
  out->blocks_streamed_out = static_cast<int64_t>(v->h_alloc->total_streamed_out);
  out->sphere_relocations = v->relocations;
  out->block_count = v->h_alloc->n_live;
  out->active_count = v->has_center ? static_cast<int64_t>(v->h_u64[0]) : 0;
  out->has_center = v->has_center ? 1 : 0;
  std::memcpy(out->last_center, v->center, sizeof(v->center));
  return RF_OK;
}

// save_volume's records, streamed: blocks in sorted coordinate order
// (volume.py:399-401), [first, first + count) of them per call.
rf_status rf_snapshot_records(rf_volume* v, int64_t first, int64_t count, void* records_host,
                              int64_t* total) {
  if (!v || !total || first < 0 || count < 0) return RF_INVALID_ARG;
  cudaSetDevice(v->cfg.device);
  cudaStream_t st = v->stream;
  int* d_list = nullptr;
  RF_CUDA_TRY(v, cudaMallocAsync(&d_list, sizeof(int) * v->T.capacity, st));
  cudaMemsetAsync(v->d_u64, 0, sizeof(unsigned long long), st);
  k_list_live<<<v->n_sms * 4, 256, 0, st>>>(v->T, d_list, v->d_u64);
  cudaMemcpyAsync(v->h_u64, v->d_u64, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
  RF_CUDA_TRY(v, cudaStreamSynchronize(st));
  const long long n = static_cast<long long>(v->h_u64[0]);
  *total = n;
  const long long m = std::max(0LL, std::min<long long>(count, n - first));
  rf_status rs = RF_OK;
  if (records_host && m > 0) {
    long long *keys = nullptr, *keys_sorted = nullptr;
    int* slots_sorted = nullptr;
    unsigned* rec = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, (long long*)nullptr, (long long*)nullptr,
                                    (int*)nullptr, (int*)nullptr, static_cast<int>(n), 0, 63, st);
    if (cudaMallocAsync(&keys, sizeof(long long) * n, st) != cudaSuccess ||
        cudaMallocAsync(&keys_sorted, sizeof(long long) * n, st) != cudaSuccess ||
        cudaMallocAsync(&slots_sorted, sizeof(int) * n, st) != cudaSuccess ||
        cudaMallocAsync(&tmp, tmp_bytes, st) != cudaSuccess ||
        cudaMallocAsync(&rec, sizeof(unsigned) * kSnapRecordWords * m, st) != cudaSuccess) {
      rs = RF_CAPACITY;
    } else {
      k_gather_keys<<<static_cast<int>((n + 255) / 256), 256, 0, st>>>(v->T, d_list, n, keys);
      cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys_sorted, d_list, slots_sorted,
                                      static_cast<int>(n), 0, 63, st);
      k_snapshot_records<<<static_cast<int>(std::min<long long>(m, v->n_sms * 16)), 256, 0, st>>>(
          v->T, slots_sorted, first, m, rec);
      cudaMemcpyAsync(records_host, rec, sizeof(unsigned) * kSnapRecordWords * m,
                      cudaMemcpyDeviceToHost, st);
    }
    for (void* p : {(void*)keys, (void*)keys_sorted, (void*)slots_sorted, (void*)rec, tmp})
      if (p) cudaFreeAsync(p, st);
  }
  cudaFreeAsync(d_list, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return fail(v, RF_CUDA, "snapshot records failed");
  if (rs != RF_OK) return fail(v, rs, "snapshot records: device memory");
  return RF_OK;
}

rf_status rf_export_blocks(rf_volume* v, int64_t* keys_host, double* data_host, int64_t cap,
                           int64_t* n_out) {
  if (!v || !n_out) return RF_INVALID_ARG;
  cudaSetDevice(v->cfg.device);
  int* d_list = nullptr;
  RF_CUDA_TRY(v, cudaMallocAsync(&d_list, sizeof(int) * v->T.capacity, v->stream));
  cudaMemsetAsync(v->d_u64, 0, sizeof(unsigned long long), v->stream);
  k_list_live<<<v->n_sms * 4, 256, 0, v->stream>>>(v->T, d_list, v->d_u64);
  cudaMemcpyAsync(v->h_u64, v->d_u64, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                  v->stream);
  RF_CUDA_TRY(v, cudaStreamSynchronize(v->stream));
  const long long n = static_cast<long long>(v->h_u64[0]);
  *n_out = n;
  if (keys_host && data_host && n > 0) {
    const long long m = std::min<long long>(n, cap);
    const long long chunk = 16384;  // bound the staging buffer (16k blocks = 335 MB)
    long long* d_keys = nullptr;
    double* d_data = nullptr;
    const long long c = std::min(chunk, m);
    RF_CUDA_TRY(v, cudaMallocAsync(&d_keys, sizeof(long long) * c, v->stream));
    RF_CUDA_TRY(v, cudaMallocAsync(&d_data, sizeof(double) * kBlockDoubles * c, v->stream));
    for (long long off = 0; off < m; off += c) {
      const long long k = std::min(c, m - off);
      k_gather<<<static_cast<int>(std::min<long long>(k, v->n_sms * 8)), 256, 0, v->stream>>>(
          v->T, d_list + off, k, d_keys, d_data);
      cudaMemcpyAsync(keys_host + off, d_keys, sizeof(long long) * k, cudaMemcpyDeviceToHost,
                      v->stream);
      cudaMemcpyAsync(data_host + off * kBlockDoubles, d_data, sizeof(double) * kBlockDoubles * k,
                      cudaMemcpyDeviceToHost, v->stream);
    }
    cudaFreeAsync(d_keys, v->stream);
    cudaFreeAsync(d_data, v->stream);
  }
  cudaFreeAsync(d_list, v->stream);
  RF_CUDA_TRY(v, cudaStreamSynchronize(v->stream));
  return RF_OK;
}


// ---- marching cubes (meshing.py:216-245) ----------------------------------

}  // extern "C"

namespace {

// Device weld of (dv, dc, dt) (meshing.py:248-276); on success the outputs
// replace the inputs (caller frees the returned buffers).
rf_status weld_device(rf_volume* v, double tol, double*& dv, double*& dc, long long*& dt,
                      long long& nv, long long& nt) {
  cudaStream_t st = v->stream;
  if (nv >= (1LL << 31) || nt >= (1LL << 31)) return RF_CAPACITY;
  const int n = static_cast<int>(nv), m = static_cast<int>(nt);
  const int g = v->n_sms * 8;
  long long *kx, *ky, *kz, *kg, *ks, *tr, *to;
  int *ia, *ib, *flag, *seg, *inv, *keep, *pos;
  double *vo, *co;
  void* tmp = nullptr;
  size_t t_sort = 0, t_scan = 0, t_scan2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t_sort, (long long*)nullptr, (long long*)nullptr,
                                  (int*)nullptr, (int*)nullptr, n, 0, 64, st);
  cub::DeviceScan::InclusiveSum(nullptr, t_scan, (int*)nullptr, (int*)nullptr, n, st);
  cub::DeviceScan::InclusiveSum(nullptr, t_scan2, (int*)nullptr, (int*)nullptr, std::max(m, 1), st);
  const size_t bn = sizeof(long long) * n;
  void** bufs[] = {(void**)&kx, (void**)&ky, (void**)&kz, (void**)&kg, (void**)&ks};
  for (void** b : bufs) RF_CUDA_TRY(v, cudaMallocAsync(b, bn, st));
  for (int** b : {&ia, &ib, &flag, &seg, &inv}) RF_CUDA_TRY(v, cudaMallocAsync(b, sizeof(int) * n, st));
  RF_CUDA_TRY(v, cudaMallocAsync(&keep, sizeof(int) * std::max(m, 1), st));
  RF_CUDA_TRY(v, cudaMallocAsync(&pos, sizeof(int) * std::max(m, 1), st));
  RF_CUDA_TRY(v, cudaMallocAsync(&tr, sizeof(long long) * 3 * std::max(m, 1), st));
  RF_CUDA_TRY(v, cudaMallocAsync(&tmp, std::max({t_sort, t_scan, t_scan2}), st));
  size_t tb = std::max({t_sort, t_scan, t_scan2});
  k_weld_keys<<<g, 256, 0, st>>>(dv, n, tol, kx, ky, kz, ia);
  // stable LSD: z, then y, then x -- lexicographic (x, y, z), ties by index
  cub::DeviceRadixSort::SortPairs(tmp, tb, kz, ks, ia, ib, n, 0, 64, st);
  k_weld_gather<<<g, 256, 0, st>>>(ky, ib, n, kg);
  tb = std::max({t_sort, t_scan, t_scan2});
  cub::DeviceRadixSort::SortPairs(tmp, tb, kg, ks, ib, ia, n, 0, 64, st);
  k_weld_gather<<<g, 256, 0, st>>>(kx, ia, n, kg);
  tb = std::max({t_sort, t_scan, t_scan2});
  cub::DeviceRadixSort::SortPairs(tmp, tb, kg, ks, ia, ib, n, 0, 64, st);
  k_weld_flags<<<g, 256, 0, st>>>(kx, ky, kz, ib, n, flag);
  tb = std::max({t_sort, t_scan, t_scan2});
  cub::DeviceScan::InclusiveSum(tmp, tb, flag, seg, n, st);
  int nu = 0, nk = 0;
  cudaMemcpyAsync(&nu, seg + (n - 1), sizeof(int), cudaMemcpyDeviceToHost, st);
  RF_CUDA_TRY(v, cudaStreamSynchronize(st));
  RF_CUDA_TRY(v, cudaMallocAsync(&vo, sizeof(double) * 3 * nu, st));
  RF_CUDA_TRY(v, cudaMallocAsync(&co, sizeof(double) * 3 * nu, st));
  k_weld_scatter<<<g, 256, 0, st>>>(ib, flag, seg, n, dv, dc, vo, co, inv);
  if (m > 0) {
    k_weld_tris<<<g, 256, 0, st>>>(dt, m, inv, tr, keep);
    tb = std::max({t_sort, t_scan, t_scan2});
    cub::DeviceScan::InclusiveSum(tmp, tb, keep, pos, m, st);
    cudaMemcpyAsync(&nk, pos + (m - 1), sizeof(int), cudaMemcpyDeviceToHost, st);
    RF_CUDA_TRY(v, cudaStreamSynchronize(st));
  }
  RF_CUDA_TRY(v, cudaMallocAsync(&to, sizeof(long long) * 3 * std::max(nk, 1), st));
  if (m > 0) k_weld_compact<<<g, 256, 0, st>>>(tr, keep, pos, m, to);
  for (void* p : {(void*)kx, (void*)ky, (void*)kz, (void*)kg, (void*)ks, (void*)ia, (void*)ib,
                  (void*)flag, (void*)seg, (void*)inv, (void*)keep, (void*)pos, (void*)tr, tmp,
                  (void*)dv, (void*)dc, (void*)dt})
    cudaFreeAsync(p, st);
  dv = vo;
  dc = co;
  dt = to;
  nv = nu;
  nt = nk;
  return RF_OK;
}

// marching_cubes (+ optional device weld when tol > 0) into host arrays.
// The peer tables marching cubes reads cross-shard neighbours from: every
// shard once connected (own entry = this table), else this table alone.
MeshPeers mesh_peers_of(const rf_volume* v) {
  MeshPeers mp = v->mesh;
  if (mp.count < 2) {
    mp.count = 1;
    mp.self = 0;
  }
  return mp;
}

rf_status mesh_to_host(rf_volume* v, double tol, double* vertices, double* colors,
                       int64_t* triangles, int64_t vcap, int64_t tcap, int64_t* nv_out,
                       int64_t* nt_out) {
  if (!v || !nv_out || !nt_out || vcap < 0 || tcap < 0) return RF_INVALID_ARG;
  cudaSetDevice(v->cfg.device);
  cudaStream_t st = v->stream;
  // every block, both tiers (meshing.py:229-231), sorted by key = by coordinate
  int* d_list = nullptr;
  RF_CUDA_TRY(v, cudaMallocAsync(&d_list, sizeof(int) * v->T.capacity, st));
  cudaMemsetAsync(v->d_u64, 0, sizeof(unsigned long long), st);
  k_list_live<<<v->n_sms * 4, 256, 0, st>>>(v->T, d_list, v->d_u64);
  cudaMemcpyAsync(v->h_u64, v->d_u64, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
  RF_CUDA_TRY(v, cudaStreamSynchronize(st));
  const long long n = static_cast<long long>(v->h_u64[0]);
  *nv_out = 0;
  *nt_out = 0;
  if (n == 0) {
    cudaFreeAsync(d_list, st);
    RF_CUDA_TRY(v, cudaStreamSynchronize(st));
    return RF_OK;
  }
  long long *keys = nullptr, *keys_sorted = nullptr, *cnt = nullptr, *off = nullptr;
  int* slots_sorted = nullptr;
  RF_CUDA_TRY(v, cudaMallocAsync(&keys, sizeof(long long) * n, st));
  RF_CUDA_TRY(v, cudaMallocAsync(&keys_sorted, sizeof(long long) * n, st));
  RF_CUDA_TRY(v, cudaMallocAsync(&slots_sorted, sizeof(int) * n, st));
  RF_CUDA_TRY(v, cudaMallocAsync(&cnt, sizeof(long long) * 2 * (n + 1), st));
  RF_CUDA_TRY(v, cudaMallocAsync(&off, sizeof(long long) * 2 * (n + 1), st));
  k_gather_keys<<<static_cast<int>((n + 255) / 256), 256, 0, st>>>(v->T, d_list, n, keys);
  size_t tmp_sort = 0, tmp_scan = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_sort, keys, keys_sorted, d_list, slots_sorted,
                                  static_cast<int>(n), 0, 63, st);
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_scan, cnt, off, static_cast<int>(n + 1), st);
  void* tmp = nullptr;
  RF_CUDA_TRY(v, cudaMallocAsync(&tmp, std::max(tmp_sort, tmp_scan), st));
  cub::DeviceRadixSort::SortPairs(tmp, tmp_sort, keys, keys_sorted, d_list, slots_sorted,
                                  static_cast<int>(n), 0, 63, st);
  // per-block counts -> exclusive offsets (entry n holds the totals)
  long long* nv = cnt;
  long long* nt = cnt + (n + 1);
  cudaMemsetAsync(cnt, 0, sizeof(long long) * 2 * (n + 1), st);
  const int grid = static_cast<int>(std::min<long long>(n, 1LL << 20));
  k_mesh_count<<<grid, kMcThreads, 0, st>>>(v->T, mesh_peers_of(v), keys_sorted, slots_sorted, n, nv, nt);
  cub::DeviceScan::ExclusiveSum(tmp, tmp_scan, nv, off, static_cast<int>(n + 1), st);
  cub::DeviceScan::ExclusiveSum(tmp, tmp_scan, nt, off + (n + 1), static_cast<int>(n + 1), st);
  long long tot[2] = {0, 0};
  cudaMemcpyAsync(&tot[0], off + n, sizeof(long long), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&tot[1], off + (n + 1) + n, sizeof(long long), cudaMemcpyDeviceToHost, st);
  rf_status rs = RF_OK;
  if (cudaStreamSynchronize(st) != cudaSuccess) rs = RF_CUDA;
  *nv_out = tot[0];
  *nt_out = tot[1];
  const bool arrays = vertices && colors && triangles;
  // unwelded sizes are known now; a welded mesh is sized by running the weld
  if (rs == RF_OK && tot[0] > 0 && (tol > 0.0 || (arrays && tot[0] <= vcap && tot[1] <= tcap))) {
    double *dv = nullptr, *dc = nullptr;
    long long* dt = nullptr;
    if (cudaMallocAsync(&dv, sizeof(double) * 3 * tot[0], st) != cudaSuccess ||
        cudaMallocAsync(&dc, sizeof(double) * 3 * tot[0], st) != cudaSuccess ||
        cudaMallocAsync(&dt, sizeof(long long) * 3 * std::max(tot[1], 1LL), st) != cudaSuccess) {
      rs = RF_CAPACITY;
    } else {
      k_mesh_emit<<<grid, kMcThreads, 0, st>>>(v->T, mesh_peers_of(v), keys_sorted, slots_sorted, n, off,
                                               off + (n + 1), v->cfg.voxel_size, dv, dc, dt);
      long long mv = tot[0], mt = tot[1];
      if (tol > 0.0) {
        rs = weld_device(v, tol, dv, dc, dt, mv, mt);
        *nv_out = mv;
        *nt_out = mt;
      }
      if (rs == RF_OK && arrays && mv <= vcap && mt <= tcap) {
        cudaMemcpyAsync(vertices, dv, sizeof(double) * 3 * mv, cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(colors, dc, sizeof(double) * 3 * mv, cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(triangles, dt, sizeof(long long) * 3 * mt, cudaMemcpyDeviceToHost, st);
      }
    }
    if (dv) cudaFreeAsync(dv, st);
    if (dc) cudaFreeAsync(dc, st);
    if (dt) cudaFreeAsync(dt, st);
  }
  for (void* p : {static_cast<void*>(d_list), static_cast<void*>(keys),
                  static_cast<void*>(keys_sorted), static_cast<void*>(slots_sorted),
                  static_cast<void*>(cnt), static_cast<void*>(off), tmp})
    cudaFreeAsync(p, st);
  if (cudaStreamSynchronize(st) != cudaSuccess || cudaGetLastError() != cudaSuccess)
    return fail(v, RF_CUDA, "marching cubes failed");
  if (rs == RF_CAPACITY) return fail(v, RF_CAPACITY, "marching cubes: device memory for the mesh");
  return rs;
}

}  // namespace

extern "C" {

rf_status rf_marching_cubes(rf_volume* v, double* vertices, double* colors, int64_t* triangles,
                            int64_t vcap, int64_t tcap, int64_t* nv_out, int64_t* nt_out) {
  return mesh_to_host(v, 0.0, vertices, colors, triangles, vcap, tcap, nv_out, nt_out);
}

rf_status rf_marching_cubes_welded(rf_volume* v, double tol, double* vertices, double* colors,
                                   int64_t* triangles, int64_t vcap, int64_t tcap,
                                   int64_t* nv_out, int64_t* nt_out) {
  if (!(tol > 0.0)) return RF_INVALID_ARG;
  return mesh_to_host(v, tol, vertices, colors, triangles, vcap, tcap, nv_out, nt_out);
}

// ---- nn_min_d2 (_kernels_cy.pyx:111-129), the plugin's evaluation kernel ----

rf_status rf_nn_min_d2(const double* q, int64_t n, const double* pts, int64_t m, double* out,
                       void* stream) {
  if (n < 0 || m < 0 || (n > 0 && (!q || !out)) || (m > 0 && !pts)) return RF_INVALID_ARG;
  if (n == 0) return RF_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double *dq = nullptr, *dp = nullptr, *dout = nullptr;
  const size_t bq = sizeof(double) * 3 * n, bp = sizeof(double) * 3 * std::max<int64_t>(m, 1);
  if (cudaMallocAsync(&dq, bq, st) != cudaSuccess || cudaMallocAsync(&dp, bp, st) != cudaSuccess ||
      cudaMallocAsync(&dout, sizeof(double) * n, st) != cudaSuccess) {
    cudaGetLastError();
    return RF_CAPACITY;
  }
  cudaMemcpyAsync(dq, q, bq, cudaMemcpyHostToDevice, st);
  if (m > 0) cudaMemcpyAsync(dp, pts, sizeof(double) * 3 * m, cudaMemcpyHostToDevice, st);
  const long long blocks = (n + 2 * kNnThreads - 1) / (2 * kNnThreads);
  k_nn_min_d2<<<static_cast<unsigned>(blocks), kNnThreads, 0, st>>>(dq, n, dp, m, dout);
  cudaMemcpyAsync(out, dout, sizeof(double) * n, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(dq, st);
  cudaFreeAsync(dp, st);
  cudaFreeAsync(dout, st);
  if (cudaStreamSynchronize(st) != cudaSuccess || cudaGetLastError() != cudaSuccess) return RF_CUDA;
  return RF_OK;
}

rf_status rf_import_blocks(rf_volume* v, const int64_t* keys_host, const double* data_host,
                           int64_t n) {
  if (!v || n < 0 || (n > 0 && (!keys_host || !data_host))) return RF_INVALID_ARG;
  if (n == 0) return RF_OK;
  cudaSetDevice(v->cfg.device);
  const long long chunk = 16384;
  long long* d_keys = nullptr;
  double* d_data = nullptr;
  int* d_ovf = reinterpret_cast<int*>(v->d_u64);
  const long long c = std::min<long long>(chunk, n);
  RF_CUDA_TRY(v, cudaMallocAsync(&d_keys, sizeof(long long) * c, v->stream));
  RF_CUDA_TRY(v, cudaMallocAsync(&d_data, sizeof(double) * kBlockDoubles * c, v->stream));
  cudaMemsetAsync(v->d_u64, 0, sizeof(unsigned long long), v->stream);
  for (long long off = 0; off < n; off += c) {
    const long long k = std::min(c, n - off);
    cudaMemcpyAsync(d_keys, keys_host + off, sizeof(long long) * k, cudaMemcpyHostToDevice,
                    v->stream);
    cudaMemcpyAsync(d_data, data_host + off * kBlockDoubles, sizeof(double) * kBlockDoubles * k,
                    cudaMemcpyHostToDevice, v->stream);
    k_import<<<static_cast<int>(std::min<long long>(k, v->n_sms * 8)), 256, 0, v->stream>>>(
        v->T, d_keys, d_data, k, d_ovf);
    k_fixup<<<1, 256, 0, v->stream>>>(v->T);
  }
  cudaFreeAsync(d_keys, v->stream);
  cudaFreeAsync(d_data, v->stream);
  cudaMemcpyAsync(v->h_u64, v->d_u64, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                  v->stream);
  RF_CUDA_TRY(v, cudaStreamSynchronize(v->stream));
  if (v->h_u64[0]) return fail(v, RF_CAPACITY, "import: block pool capacity exhausted");
  return RF_OK;
}

rf_status rf_read_blocks(rf_volume* v, const int64_t* keys_host, int64_t n, double* data_host,
                         int32_t* found_host) {
  if (!v || n < 0 || (n > 0 && (!keys_host || !data_host))) return RF_INVALID_ARG;
  if (n == 0) return RF_OK;
  cudaSetDevice(v->cfg.device);
  long long* d_keys = nullptr;
  long long* d_keys_out = nullptr;
  double* d_data = nullptr;
  int* d_slots = nullptr;
  RF_CUDA_TRY(v, cudaMallocAsync(&d_keys, sizeof(long long) * n, v->stream));
  RF_CUDA_TRY(v, cudaMallocAsync(&d_keys_out, sizeof(long long) * n, v->stream));
  RF_CUDA_TRY(v, cudaMallocAsync(&d_slots, sizeof(int) * n, v->stream));
  RF_CUDA_TRY(v, cudaMallocAsync(&d_data, sizeof(double) * kBlockDoubles * n, v->stream));
  cudaMemcpyAsync(d_keys, keys_host, sizeof(long long) * n, cudaMemcpyHostToDevice, v->stream);
  k_lookup<<<v->n_sms * 4, 256, 0, v->stream>>>(v->T, d_keys, n, d_slots);
  k_gather<<<static_cast<int>(std::min<long long>(n, v->n_sms * 8)), 256, 0, v->stream>>>(
      v->T, d_slots, n, d_keys_out, d_data);
  cudaMemcpyAsync(data_host, d_data, sizeof(double) * kBlockDoubles * n, cudaMemcpyDeviceToHost,
                  v->stream);
  std::vector<int> slots(static_cast<size_t>(n));
  cudaMemcpyAsync(slots.data(), d_slots, sizeof(int) * n, cudaMemcpyDeviceToHost, v->stream);
  cudaFreeAsync(d_keys, v->stream);
  cudaFreeAsync(d_keys_out, v->stream);
  cudaFreeAsync(d_slots, v->stream);
  cudaFreeAsync(d_data, v->stream);
  RF_CUDA_TRY(v, cudaStreamSynchronize(v->stream));
  if (found_host)
    for (long long i = 0; i < n; ++i) found_host[i] = slots[static_cast<size_t>(i)] >= 0;
  return RF_OK;
}

rf_status rf_fuse_block(double* d, double* w, double* c, double ox, double oy, double oz,
                        double voxel_size, const double* rot_wc, double tx, double ty, double tz,
                        double fx, double fy, double cx, double cy, int32_t width, int32_t height,
                        const double* kf_depth, const double* kf_weight, const double* kf_color,
                        double mu, double eps_w, int32_t remove, int32_t* count_out) {
  if (!d || !w || !c || !rot_wc || !kf_depth || !kf_weight || !count_out || width <= 0 ||
      height <= 0)
    return RF_INVALID_ARG;
  const size_t npix = static_cast<size_t>(width) * height;
  std::vector<double> blk(kBlockDoubles);
  for (int l = 0; l < kBlockVoxels; ++l) {
    blk[l] = d[l];
    blk[kBlockVoxels + l] = w[l];
    blk[2 * kBlockVoxels + l] = c[3 * l];
    blk[3 * kBlockVoxels + l] = c[3 * l + 1];
    blk[4 * kBlockVoxels + l] = c[3 * l + 2];
  }
  double *d_blk = nullptr, *d_kd = nullptr, *d_kw = nullptr, *d_kc = nullptr;
  int* d_cnt = nullptr;
  unsigned long long* d_def = nullptr;  // deferred-voxel list + count (512 + 1 entries)
  bool ok = cudaMalloc(&d_def, sizeof(unsigned long long) * (kBlockVoxels + 1)) == cudaSuccess &&
            cudaMalloc(&d_blk, sizeof(double) * kBlockDoubles) == cudaSuccess &&
            cudaMalloc(&d_kd, sizeof(double) * npix) == cudaSuccess &&
            cudaMalloc(&d_kw, sizeof(double) * npix) == cudaSuccess &&
            cudaMalloc(&d_cnt, sizeof(int)) == cudaSuccess &&
            (!kf_color || cudaMalloc(&d_kc, sizeof(double) * 3 * npix) == cudaSuccess);
  rf_status st = RF_OK;
  if (ok) {
    cudaMemcpy(d_blk, blk.data(), sizeof(double) * kBlockDoubles, cudaMemcpyHostToDevice);
    cudaMemcpy(d_kd, kf_depth, sizeof(double) * npix, cudaMemcpyHostToDevice);
    cudaMemcpy(d_kw, kf_weight, sizeof(double) * npix, cudaMemcpyHostToDevice);
    if (kf_color) cudaMemcpy(d_kc, kf_color, sizeof(double) * 3 * npix, cudaMemcpyHostToDevice);
    FuseParams p{};
    p.kf.depth = d_kd;
    p.kf.weight = d_kw;
    p.kf.color = d_kc;
    p.kf.width = width;
    p.kf.height = height;
    p.kf.fx = fx;
    p.kf.fy = fy;
    p.kf.cx = cx;
    p.kf.cy = cy;
    std::memcpy(p.Rwc, rot_wc, sizeof(p.Rwc));
    p.t[0] = tx;
    p.t[1] = ty;
    p.t[2] = tz;
    p.voxel_size = voxel_size;
    p.mu = mu;
    p.eps_w = eps_w;
    set_dim_bits(p);
    int cnt = 0;
    unsigned* d_defn = reinterpret_cast<unsigned*>(d_def + kBlockVoxels);
    cudaMemset(d_defn, 0, sizeof(unsigned));
    if (remove) {
      k_fuse_single<kCheckRemove><<<1, kFuseThreads>>>(p, d_blk, ox, oy, oz, d_cnt,
                                                                        d_def, d_defn);
      cudaMemcpy(&cnt, d_cnt, sizeof(int), cudaMemcpyDeviceToHost);
      if (cnt == 0) {
        cudaMemset(d_defn, 0, sizeof(unsigned));
        k_fuse_single<kApplyRemove><<<1, kFuseThreads>>>(p, d_blk, ox, oy, oz,
                                                                          d_cnt, d_def, d_defn);
        cudaMemcpy(&cnt, d_cnt, sizeof(int), cudaMemcpyDeviceToHost);
      }
    } else {
      k_fuse_single<kIntegrate><<<1, kFuseThreads>>>(p, d_blk, ox, oy, oz, d_cnt,
                                                                      d_def, d_defn);
      cudaMemcpy(&cnt, d_cnt, sizeof(int), cudaMemcpyDeviceToHost);
    }
    if (cudaDeviceSynchronize() != cudaSuccess || cudaGetLastError() != cudaSuccess) {
      st = RF_CUDA;
    } else {
      cudaMemcpy(blk.data(), d_blk, sizeof(double) * kBlockDoubles, cudaMemcpyDeviceToHost);
      for (int l = 0; l < kBlockVoxels; ++l) {
        d[l] = blk[l];
        w[l] = blk[kBlockVoxels + l];
        c[3 * l] = blk[2 * kBlockVoxels + l];
        c[3 * l + 1] = blk[3 * kBlockVoxels + l];
        c[3 * l + 2] = blk[4 * kBlockVoxels + l];
      }
      *count_out = cnt;
    }
  } else {
    st = RF_CUDA;
  }
  cudaFree(d_def);
  cudaFree(d_blk);
  cudaFree(d_kd);
  cudaFree(d_kw);
  cudaFree(d_kc);
  cudaFree(d_cnt);
  return st;
}

rf_status rf_selftest_division(uint64_t n, uint64_t seed, int32_t exp_span, uint64_t* mismatches) {
  if (!mismatches || exp_span < 0 || exp_span > 1000) return RF_INVALID_ARG;
  unsigned long long* d = nullptr;
  if (cudaMalloc(&d, sizeof(unsigned long long)) != cudaSuccess) return RF_CUDA;
  cudaMemset(d, 0, sizeof(unsigned long long));
  k_selftest_division<<<148 * 8, 256>>>(n, seed, exp_span, d);
  unsigned long long h = 0;
  cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const cudaError_t e = cudaGetLastError();
  cudaFree(d);
  if (e != cudaSuccess) return RF_CUDA;
  *mismatches = h;
  return RF_OK;
}

rf_status rf_selftest_projection(int32_t width, int32_t height, double cx, double cy,
                                 uint64_t n, uint64_t seed, uint64_t* mismatches) {
  if (!mismatches || width <= 0 || height <= 0) return RF_INVALID_ARG;
  FuseParams p{};
  p.kf.width = width;
  p.kf.height = height;
  p.kf.cx = cx;
  p.kf.cy = cy;
  set_dim_bits(p);
  if (!p.fast_proj) return RF_INVALID_ARG;
  unsigned long long* d = nullptr;
  if (cudaMalloc(&d, sizeof(unsigned long long)) != cudaSuccess) return RF_CUDA;
  cudaMemset(d, 0, sizeof(unsigned long long));
  k_selftest_projection<<<148 * 8, 256>>>(p, n, seed, d);
  unsigned long long h = 0;
  cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const cudaError_t e = cudaGetLastError();
  cudaFree(d);
  if (e != cudaSuccess) return RF_CUDA;
  *mismatches = h;
  return RF_OK;
}

rf_status rf_set_memo_budget(rf_volume* v, int64_t bytes) {
  if (!v || bytes < 0) return RF_INVALID_ARG;
  cudaSetDevice(v->cfg.device);
  memo_release(v);  // slots are re-carved for the new budget at next use
  v->memo_budget = static_cast<size_t>(bytes);
  return RF_OK;
}

rf_status rf_profile_begin(rf_volume* v) {
  if (!v) return RF_INVALID_ARG;
  for (auto& e : v->events) {
    v->event_pool.push_back(e.a);
    v->event_pool.push_back(e.b);
  }
  v->events.clear();
  v->prof_voxels = v->prof_pixels = v->prof_blocks = v->prof_launches = 0;
  v->prof_int_vox = v->prof_int_pix = v->prof_rem_vox = v->prof_rem_pix = 0;
  v->prof_rem_ops = 0;
  v->profiling = true;
  return RF_OK;
}

rf_status rf_profile_end(rf_volume* v, rf_profile* out) {
  if (!v || !out) return RF_INVALID_ARG;
  cudaSetDevice(v->cfg.device);
  RF_CUDA_TRY(v, cudaStreamSynchronize(v->stream));
  rf_profile p{};
  for (auto& e : v->events) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e.a, e.b);
    if (e.kind == 0 || e.kind == 4) {  // 0 integrate, 4 the removal pass
      p.fuse_launches++;
      p.fuse_ms += ms;
      if (e.kind == 0) {
        p.integrate_launches++;
        p.integrate_ms += ms;
      } else {
        p.removal_ms += ms;
      }
    } else if (e.kind == 1) {  // the removal's check (k_check)
      p.check_launches++;
      p.check_ms += ms;
      p.removal_ms += ms;
    } else if (e.kind == 2) {
      p.footprint_launches++;
      p.footprint_ms += ms;
    } else {
      p.other_launches++;
      p.other_ms += ms;
    }
    v->event_pool.push_back(e.a);
    v->event_pool.push_back(e.b);
  }
  v->events.clear();
  p.voxels_updated = v->prof_voxels;
  p.pixels = v->prof_pixels;
  p.blocks_touched = v->prof_blocks;
  p.kernel_launches = v->prof_launches;
  p.integrate_voxels = v->prof_int_vox;
  p.integrate_pixels = v->prof_int_pix;
  p.removal_ops = v->prof_rem_ops;
  p.removal_voxels = v->prof_rem_vox;
  p.removal_pixels = v->prof_rem_pix;
  v->profiling = false;
  *out = p;
  return RF_OK;
}

}  // extern "C"

// ---- cross-shard marching cubes --------------------------------

extern "C" {

rf_status rf_mesh_connect(rf_volume* v, rf_volume* const* shards, int32_t count) {
  if (!v || !shards || count != v->cfg.shard_count || count < 2 || count > kMaxShards)
    return RF_INVALID_ARG;
  if (shards[v->cfg.shard_rank] != v)
    return fail(v, RF_INVALID_ARG, "rf_mesh_connect: own entry mismatch");
  MeshPeers mp{};
  for (int s = 0; s < count; ++s) {
    const rf_volume* o = shards[s];
    if (!o || o->cfg.shard_count != count || o->cfg.shard_rank != s) return RF_INVALID_ARG;
    mp.p[s] = MeshPeer{o->T.heads, o->T.keys, o->T.next, o->T.pool, o->T.buckets};
  }
  mp.count = count;
  mp.self = v->cfg.shard_rank;
  v->mesh = mp;
  return RF_OK;
}

rf_status rf_mesh_ipc_handle(rf_volume* v, void* handles) {
  if (!v || !handles) return RF_INVALID_ARG;
  cudaSetDevice(v->cfg.device);
  const void* arr[4] = {v->T.heads, v->T.keys, v->T.next, v->T.pool};
  for (int a = 0; a < 4; ++a) {
    cudaIpcMemHandle_t h;
    RF_CUDA_TRY(v, cudaIpcGetMemHandle(&h, const_cast<void*>(arr[a])));
    std::memcpy(static_cast<char*>(handles) + a * sizeof(h), &h, sizeof(h));
  }
  return RF_OK;
}

rf_status rf_mesh_ipc_open(rf_volume* v, const void* handles, const int64_t* buckets) {
  if (!v || !handles || !buckets || v->cfg.shard_count < 2) return RF_INVALID_ARG;
  cudaSetDevice(v->cfg.device);
  const int G = v->cfg.shard_count;
  MeshPeers mp{};
  for (int s = 0; s < G; ++s) {
    if (s == v->cfg.shard_rank) {
      mp.p[s] = MeshPeer{v->T.heads, v->T.keys, v->T.next, v->T.pool, v->T.buckets};
      continue;
    }
    void* ptr[4] = {};
    for (int a = 0; a < 4; ++a) {
      if (v->mesh_ipc[s][a]) {
        ptr[a] = v->mesh_ipc[s][a];
        continue;
      }
      cudaIpcMemHandle_t h;
      std::memcpy(&h, static_cast<const char*>(handles) + (4 * s + a) * sizeof(h), sizeof(h));
      RF_CUDA_TRY(v, cudaIpcOpenMemHandle(&ptr[a], h, cudaIpcMemLazyEnablePeerAccess));
      v->mesh_ipc[s][a] = ptr[a];
    }
    mp.p[s] = MeshPeer{static_cast<const int*>(ptr[0]), static_cast<const long long*>(ptr[1]),
                       static_cast<const int*>(ptr[2]), static_cast<const double*>(ptr[3]),
                       static_cast<long long>(buckets[s])};
  }
  mp.count = G;
  mp.self = v->cfg.shard_rank;
  v->mesh = mp;
  return RF_OK;
}

rf_status rf_mesh_blocks(rf_volume* v, int64_t* keys, int64_t* vcounts, int64_t* tcounts,
                         int64_t cap, int64_t* n_out) {
  if (!v || !n_out || cap < 0) return RF_INVALID_ARG;
  cudaSetDevice(v->cfg.device);
  cudaStream_t st = v->stream;
  int* d_list = nullptr;
  RF_CUDA_TRY(v, cudaMallocAsync(&d_list, sizeof(int) * v->T.capacity, st));
  cudaMemsetAsync(v->d_u64, 0, sizeof(unsigned long long), st);
  k_list_live<<<v->n_sms * 4, 256, 0, st>>>(v->T, d_list, v->d_u64);
  cudaMemcpyAsync(v->h_u64, v->d_u64, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
  RF_CUDA_TRY(v, cudaStreamSynchronize(st));
  const long long n = static_cast<long long>(v->h_u64[0]);
  *n_out = n;
  rf_status rs = RF_OK;
  if (n > 0 && keys && vcounts && tcounts && n <= cap) {
    long long *dk = nullptr, *dks = nullptr, *cnt = nullptr;
    int* slots_sorted = nullptr;
    void* tmp = nullptr;
    size_t tmp_sort = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_sort, dk, dks, d_list, slots_sorted,
                                    static_cast<int>(n), 0, 63, st);
    if (cudaMallocAsync(&dk, sizeof(long long) * n, st) != cudaSuccess ||
        cudaMallocAsync(&dks, sizeof(long long) * n, st) != cudaSuccess ||
        cudaMallocAsync(&slots_sorted, sizeof(int) * n, st) != cudaSuccess ||
        cudaMallocAsync(&cnt, sizeof(long long) * 2 * n, st) != cudaSuccess ||
        cudaMallocAsync(&tmp, std::max<size_t>(tmp_sort, 1), st) != cudaSuccess) {
      rs = RF_CAPACITY;
    } else {
      k_gather_keys<<<static_cast<int>((n + 255) / 256), 256, 0, st>>>(v->T, d_list, n, dk);
      cub::DeviceRadixSort::SortPairs(tmp, tmp_sort, dk, dks, d_list, slots_sorted,
                                      static_cast<int>(n), 0, 63, st);
      cudaMemsetAsync(cnt, 0, sizeof(long long) * 2 * n, st);
      const int grid = static_cast<int>(std::min<long long>(n, 1LL << 20));
      k_mesh_count<<<grid, kMcThreads, 0, st>>>(v->T, mesh_peers_of(v), dks, slots_sorted, n,
                                                cnt, cnt + n);
      cudaMemcpyAsync(keys, dks, sizeof(long long) * n, cudaMemcpyDeviceToHost, st);
      cudaMemcpyAsync(vcounts, cnt, sizeof(long long) * n, cudaMemcpyDeviceToHost, st);
      cudaMemcpyAsync(tcounts, cnt + n, sizeof(long long) * n, cudaMemcpyDeviceToHost, st);
    }
    for (void* b : {static_cast<void*>(dk), static_cast<void*>(dks),
                    static_cast<void*>(slots_sorted), static_cast<void*>(cnt), tmp})
      if (b) cudaFreeAsync(b, st);
  }
  cudaFreeAsync(d_list, st);
  RF_CUDA_TRY(v, cudaStreamSynchronize(st));
  return rs;
}

}  // extern "C"
