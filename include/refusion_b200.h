/*
 * refusion_b200.h -- C ABI of the B200-native surface-correction hot path.
 *
 * Drop-in boundary for the reference package `refusion` (arXiv 1709.03763):
 * the reference's plugin point is the kernel backend `refusion.kernels`
 * (src/refusion/kernels.py:19-41, selected by REFUSION_BACKEND) and the
 * volume API it serves (src/refusion/volume.py).  Every entry point below
 * names the reference function it replaces.  Paths are relative to
 * /root/reference/pkg/.
 *
 * Conventions
 *  - Plain C types only; every call returns an rf_status.
 *  - Keyframe planes (rf_kf_view) are DEVICE pointers owned by the caller;
 *    they must stay alive until the call returns (calls that return
 *    results synchronise the volume's stream; rf_stream_async does not).
 *  - Host buffers (keys, exported blocks) are plain host memory.
 *  - One volume-mutating call at a time per rf_volume; calls are
 *    ordered on the volume's CUDA stream (rf_set_cuda_stream).
 *  - Block keys pack (bx, by, bz) as ((bx+2^20)<<42)|((by+2^20)<<21)|(bz+2^20)
 *    (src/refusion/volume.py:137-148).
 *  - Exported / imported block records are 5 planes of 512 doubles:
 *    D, W, C0, C1, C2 with voxel index l = x + 8y + 64z
 *    (src/refusion/volume.py:69-81).
 */
#ifndef REFUSION_B200_H
#define REFUSION_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum rf_status {
    RF_OK = 0,
    RF_STREAMING_CONTRACT = 1,  /* errors.StreamingContractError (src/refusion/errors.py:20) */
    RF_INCONSISTENT = 2,        /* errors.VolumeInconsistencyError (src/refusion/errors.py:24) */
    RF_CAPACITY = 3,            /* block pool exhausted */
    RF_INVALID_ARG = 4,         /* ValueError */
    RF_CUDA = 5                 /* CUDA runtime failure */
} rf_status;

typedef struct rf_volume rf_volume;

/* VolumeConfig (src/refusion/volume.py:39-66) plus device sizing. */
typedef struct rf_config {
    double voxel_size;       /* metres */
    double mu;               /* truncation band */
    double stream_radius;    /* active-sphere radius */
    int64_t hash_buckets;    /* bucket count of block_hash (any > 0) */
    int64_t block_capacity;  /* max resident blocks (20,480 B each) */
    int32_t device;          /* CUDA device ordinal */
    int32_t shard_rank;      /* this GPU's shard (0 when unsharded) */
    int32_t shard_count;     /* number of shards (1 when unsharded) */
    int32_t max_pixels;      /* largest keyframe width*height (0 -> 640*480) */
} rf_config;

/* Pose (src/refusion/geometry.py:41-62): p_world = R p_cam + t, R row-major. */
typedef struct rf_pose {
    double R[9];
    double t[3];
} rf_pose;

/* Duck-typed keyframe (reference tests/test_volume.py:12-20). */
typedef struct rf_kf_view {
    const double *depth;   /* [height][width] device */
    const double *weight;  /* [height][width] device */
    const double *color;   /* [height][width][3] device, or NULL (zeros, volume.py:256-259) */
    int32_t width, height;
    double fx, fy, cx, cy;
    /* cudaEvent_t recorded after the planes' upload (e.g. on a copy stream),
     * or NULL: the volume's stream waits on it before the first kernel that
     * reads this keyframe, so host->device uploads overlap earlier entries'
     * fusion inside one batched call. */
    void *ready_event;
    /* Identity of the keyframe's planes for the footprint memo, or 0 (the
     * device pointers are the identity).  Callers uploading host planes per
     * call pass a stable tag (e.g. the host buffer's address) so that a
     * de-integration can reuse the footprint of the matching integration;
     * the memo still validates the planes by content hash. */
    uint64_t memo_tag;
    /* 1: depth / weight / color are HOST pointers (pinned for asynchronous
     * copies): the volume stages them on its copy stream into device slots,
     * each entry's kernels waiting only for its own upload, so uploads
     * overlap the fusion of earlier entries.  0: device pointers. */
    int32_t planes_on_host;
} rf_kf_view;

/* IntegrationRecord counts (src/refusion/volume.py:126-134). */
typedef struct rf_op_result {
    int64_t blocks_touched;
    int64_t voxels_updated;
    int64_t n_new;
} rf_op_result;

/* stream() return dict (src/refusion/volume.py:375-379). */
typedef struct rf_stream_result {
    int64_t streamed_in;
    int64_t streamed_out;
    int64_t relocated;
} rf_stream_result;

/* TwoTierStore counters (src/refusion/volume.py:104-110). */
typedef struct rf_counters {
    int64_t blocks_streamed_in;
    int64_t blocks_streamed_out;
    int64_t sphere_relocations;
    int64_t block_count;
    int64_t active_count;      /* blocks inside the sphere around last_center */
    int32_t has_center;
    int32_t _pad;
    double last_center[3];
} rf_counters;

/* One batched pose-graph correction (reintegration.py:156-181). */
typedef struct rf_window_result {
    int32_t status;          /* rf_status of the window */
    int32_t failed_entry;    /* entry index that raised, -1 if none */
    int32_t failed_phase;    /* 0 de-integration, 1 integration, -1 none */
    int32_t failed_window;   /* window index that raised (rf_correct_windows), -1 if none */
    int64_t n_corrected;     /* entries re-integrated (0 on error) */
    int64_t voxels_updated;  /* summed over the integrate phase */
    int64_t blocks_touched;  /* summed over all (de)integrations */
    int64_t n_new;           /* blocks allocated during the window */
    int64_t gc_freed;        /* blocks dropped by the closing GC */
} rf_window_result;

/* Device-side timing of the hot kernels (CUDA events on the volume's stream). */
typedef struct rf_profile {
    int64_t fuse_launches;       /* integrate/de-integrate apply kernels */
    double fuse_ms;              /* summed device time of those launches */
    int64_t check_launches;      /* de-integration check kernels */
    double check_ms;
    int64_t footprint_launches;  /* footprint + allocation kernels */
    double footprint_ms;
    int64_t voxels_updated;      /* voxels written by profiled fuse launches */
    int64_t pixels;              /* keyframe pixels read by profiled fuse launches */
    int64_t blocks_touched;
    int64_t kernel_launches;     /* every kernel this library launched while profiling */
    int64_t other_launches;      /* streaming, GC and bookkeeping kernels */
    double other_ms;
    /* per operation: integrations (k_fuse<kIntegrate>) and de-integrations
     * (the check k_check + the removal k_fuse<kApplyRemove>) */
    int64_t integrate_launches;
    double integrate_ms;
    int64_t integrate_voxels;
    int64_t integrate_pixels;
    int64_t removal_ops;
    double removal_ms;
    int64_t removal_voxels;
    int64_t removal_pixels;
} rf_profile;

/* ---- lifecycle ------------------------------------------------------- */
/* TwoTierStore() (volume.py:96-110) */
rf_status rf_volume_create(const rf_config *cfg, rf_volume **out);
rf_status rf_volume_destroy(rf_volume *vol);
/* stream is a cudaStream_t (NULL = legacy default stream) */
rf_status rf_set_cuda_stream(rf_volume *vol, void *stream);
const char *rf_last_error(const rf_volume *vol);
const char *rf_status_string(int status);

/* ---- hashing ----------------------------------------------------------- */
/* block_hash (volume.py:84-93): XOR of prime products, floor-mod buckets */
int64_t rf_block_hash(int64_t x, int64_t y, int64_t z, int64_t buckets);
/* shard owning a packed key (multi-GPU hash sharding) */
int32_t rf_key_owner(int64_t key, int32_t shard_count);

/* ---- volume operations --------------------------------------------- */
/* stream (volume.py:351-379).  result may be NULL: then nothing syncs. */
rf_status rf_stream(rf_volume *vol, const double center[3], rf_stream_result *result);
/* keyframe_block_footprint (volume.py:151-197): sorted unique keys, no allocation.
 * *n_out receives the count; if it exceeds cap nothing is written past cap. */
rf_status rf_footprint(rf_volume *vol, const rf_kf_view *kf, const rf_pose *pose,
                       int64_t *keys_host, int64_t cap, int64_t *n_out);
/* allocate_blocks (volume.py:216-249): new keys (unsorted) into keys_host. */
rf_status rf_allocate(rf_volume *vol, const rf_kf_view *kf, const rf_pose *pose,
                      int64_t *new_keys_host, int64_t cap, int64_t *n_new);
/* integrate (volume.py:296-312); new_keys_host may be NULL. */
rf_status rf_integrate(rf_volume *vol, const rf_kf_view *kf, const rf_pose *pose,
                       rf_op_result *result, int64_t *new_keys_host, int64_t new_cap);
/* deintegrate (volume.py:315-338); all-or-nothing as the reference. */
rf_status rf_deintegrate(rf_volume *vol, const rf_kf_view *kf, const rf_pose *pose,
                         rf_op_result *result);
/* reintegration._correct_entries (reintegration.py:156-181) for m entries,
 * followed by stream(next_center) when next_center != NULL
 * (correct_window / correct_topk, reintegration.py:184-209).  One host
 * synchronisation per call. */
rf_status rf_correct(rf_volume *vol, int32_t m, const rf_kf_view *kfs,
                     const rf_pose *old_poses, const rf_pose *new_poses,
                     const double *next_center, rf_window_result *result);
/* n_windows back-to-back _correct_entries calls (correct_topk's one window
 * per pick, finalize's runs of m) in one batch with ONE host sync: window w
 * holds sizes[w] consecutive entries of kfs / old_poses / new_poses.  On an
 * error the windows before the failing one stay applied (as sequential
 * calls would leave them) and result->failed_window names it. */
rf_status rf_correct_windows(rf_volume *vol, int32_t n_windows, const int32_t *sizes,
                             const rf_kf_view *kfs, const rf_pose *old_poses,
                             const rf_pose *new_poses, const double *next_center,
                             rf_window_result *result);
/* garbage_collect (volume.py:382-390) */
rf_status rf_garbage_collect(rf_volume *vol, int64_t *freed);
/* total_weight (volume.py:393-394) */
rf_status rf_total_weight(rf_volume *vol, double *out);
rf_status rf_counters_get(rf_volume *vol, rf_counters *out);

/* ---- snapshots / parity (volume.py:397-464) --------------------------- */
/* keys [n], data [n][5][512] doubles (D, W, C0, C1, C2); slot order. */
rf_status rf_export_blocks(rf_volume *vol, int64_t *keys_host, double *data_host,
                           int64_t cap, int64_t *n_out);
/* marching_cubes (meshing.py:216-245) on the device: vertices and colors
 * [nv][3] doubles, triangles [nt][3] int64, in the reference's order (blocks
 * by sorted coordinate, cells by voxel index, cut edges by edge index).
 * *nv / *nt always receive the sizes; the arrays are written only when all
 * three are non-NULL and large enough (call once with NULL to size them). */
rf_status rf_marching_cubes(rf_volume *vol, double *vertices, double *colors, int64_t *triangles,
                            int64_t vcap, int64_t tcap, int64_t *nv, int64_t *nt);
/* marching_cubes followed by weld(mesh, tol) (meshing.py:248-276), both on the
 * device: the welded mesh only crosses to the host.  Same sizing protocol. */
rf_status rf_marching_cubes_welded(rf_volume *vol, double tol, double *vertices, double *colors,
                                   int64_t *triangles, int64_t vcap, int64_t tcap, int64_t *nv,
                                   int64_t *nt);
/* Cross-shard marching cubes (meshing.py:112-147 borrows the +x/+y/+z
 * neighbour blocks): on a hash-sharded volume a neighbour may be owned by
 * another shard; once connected, each shard's marching cubes reads those
 * neighbours' corners from the owner's pool (same device, or NVLink peers
 * mapped by CUDA IPC), so the union of the shards' meshes is the unsharded
 * mesh.  rf_mesh_connect: in-process shards (shards[rank] == vol).
 * rf_mesh_ipc_handle: this shard's four table allocations (heads, keys,
 * next, pool) as 4 cudaIpcMemHandle_t (256 bytes).  rf_mesh_ipc_open: every
 * shard's 4 handles [count][4] (own entry ignored) and hash_buckets. */
rf_status rf_mesh_connect(rf_volume *vol, rf_volume *const *shards, int32_t count);
rf_status rf_mesh_ipc_handle(rf_volume *vol, void *handles);
rf_status rf_mesh_ipc_open(rf_volume *vol, const void *handles, const int64_t *buckets);
/* The per-block layout of rf_marching_cubes' output: the store's block keys
 * in sorted order with each block's vertex / triangle counts (to merge the
 * shards' meshes into the unsharded order).  Sizing protocol as above. */
rf_status rf_mesh_blocks(rf_volume *vol, int64_t *keys, int64_t *vcounts, int64_t *tcounts,
                         int64_t cap, int64_t *n_out);
/* nn_min_d2 (_kernels_cy.pyx:111-129; refusion.kernels.nn_min_d2): out[i] =
 * min_j (dx*dx + dy*dy) + dz*dz over pts, q [n][3] / pts [m][3] / out [n]
 * HOST arrays (copied through the device); +inf when m == 0.  stream may be
 * NULL.  Needs no volume. */
rf_status rf_nn_min_d2(const double *q, int64_t n, const double *pts, int64_t m, double *out,
                       void *stream);

/* ---- evaluation: exact nearest-neighbour grid index ------
 * GridIndex of /root/reference/pkg/src/refusion/evaluation.py:108-229 on the
 * device: points bucketed into cells of cell_size (floor(p / cell_size),
 * packed like _pack_cells), queries scan rings of cells outward and fall
 * back to the exact linear scan exactly where the reference does; every
 * distance is the IEEE sqrt of the exact minimum of (dx*dx + dy*dy) + dz*dz
 * over the indexed points, bit-identical to the reference.  points, queries
 * and out are DEVICE pointers ([n][3], [m][3], [m] f64); the index owns a
 * sorted copy of the points. */
typedef struct rf_grid_index rf_grid_index;
rf_status rf_grid_index_create(const double *points, int64_t n, double cell_size,
                               rf_grid_index **index, void *stream);
rf_status rf_grid_index_query(rf_grid_index *index, const double *queries, int64_t m,
                              double *out, void *stream);
rf_status rf_grid_index_destroy(rf_grid_index *index);
/* save_volume's SDFV1 records (volume.py:397-415), streamed: records_host
 * receives blocks [first, first + count) in sorted coordinate order, each
 * 3 x int32 coordinate + 512 x 5 f64 (D, W, C0, C1, C2 per voxel) = 20,492 B,
 * byte-identical to the reference's file body; *total = block count
 * (records_host may be NULL to query it). */
rf_status rf_snapshot_records(rf_volume *vol, int64_t first, int64_t count, void *records_host,
                              int64_t *total);
/* insert blocks with the given contents (load_volume, volume.py:418-442) */
rf_status rf_import_blocks(rf_volume *vol, const int64_t *keys_host,
                           const double *data_host, int64_t n);
/* read back selected blocks by key; missing blocks -> found[i] = 0 */
rf_status rf_read_blocks(rf_volume *vol, const int64_t *keys_host, int64_t n,
                         double *data_host, int32_t *found_host);

/* ---- the reference kernel plugin point --------------------------------- */
/* kernels.fuse_block (src/refusion/_kernels_cy.pyx:14-108): one block, HOST
 * arrays, same argument meaning and in-place semantics; runs the same
 * device code as rf_integrate.  *count_out = voxels updated or -1. */
rf_status rf_fuse_block(double *d, double *w, double *c,
                        double ox, double oy, double oz, double voxel_size,
                        const double *rot_wc, double tx, double ty, double tz,
                        double fx, double fy, double cx, double cy,
                        int32_t width, int32_t height,
                        const double *kf_depth, const double *kf_weight,
                        const double *kf_color, double mu, double eps_w,
                        int32_t remove, int32_t *count_out);

/* Device memory the footprint memo may use (default 2 GiB; 0 disables it).
 * The memo keeps, per (keyframe planes, pose), the block keys its footprint
 * produced, so the matching de-integration skips the ray sampling; a 64-bit
 * content hash of the depth/weight planes guards against in-place edits. */
rf_status rf_set_memo_budget(rf_volume *vol, int64_t bytes);

/* ---- routed footprints (hash-sharded volumes) ---------------
 * No reference counterpart: the reference is one process (volume.py:151-249
 * is what these split across shards).  Once connected, every footprint op
 * of a shard is sampled cooperatively: rf_route makes shard r sample the
 * pixel tiles t with t mod shard_count == r and store each distinct block
 * key straight into its owner's inbox (peer memory over NVLink), then
 * synchronises.  After a barrier across the shards (the caller's:
 * torch.distributed, threads ...) the next rf_allocate / rf_integrate /
 * rf_deintegrate (1 op) or rf_correct_windows (per window: its m removal
 * footprints, then its m integration footprints) consumes those inboxes --
 * exactly that many ops, else RF_INVALID_ARG.  centers (3 per op, may be
 * NULL = the volume's current centre) is the streaming centre each op's
 * contract is checked against.  The footprint memo is off when routed. */
/* allocate this shard's inbox: max_ops footprints per call, cap_keys keys
 * per (op, sending shard); *inbox / *bytes describe the device buffer */
rf_status rf_route_setup(rf_volume *vol, int32_t max_ops, int64_t cap_keys, void **inbox,
                         uint64_t *bytes);
/* shards of one process: inboxes[s] = shard s's inbox (device pointers) */
rf_status rf_route_connect(rf_volume *vol, void *const *inboxes);
/* shards in separate processes: 64-byte cudaIpcMemHandle_t of this inbox,
 * and open all shards' handles (shard_count x 64 bytes, own entry ignored) */
rf_status rf_route_ipc_handle(rf_volume *vol, void *handle);
rf_status rf_route_ipc_open(rf_volume *vol, const void *handles);
rf_status rf_route(rf_volume *vol, int32_t n, const rf_kf_view *kfs, const rf_pose *poses,
                   const double *centers);

/* ---- cross-shard removal verdicts (hash-sharded volumes) ----
 * The reference's de-integration is all-or-nothing over the whole footprint
 * (volume.py:315-338; the window rollback reintegration.py:166-174).  Once
 * the shards are connected, every removal's check ends with a device-side
 * exchange: each shard folds its minimum failing block key into every
 * shard's slot (remote atomicMin over peer memory) and waits for all of
 * them, so every shard fails at the same op with the same global key and
 * applies the same rollback.  Calls that de-integrate (rf_deintegrate,
 * rf_correct_windows) must then be made in lockstep on every shard (the
 * callers agree on each call's status); a peer that never arrives turns
 * into RF_CAPACITY after ~60 s instead of a hang. */
/* allocate this shard's slots (max_ops ops per call); *slots / *bytes
 * describe the device buffer */
rf_status rf_shard_sync_setup(rf_volume *vol, int32_t max_ops, void **slots, uint64_t *bytes);
/* shards of one process: slots[s] = shard s's buffer (device pointers) */
rf_status rf_shard_sync_connect(rf_volume *vol, void *const *slots);
/* shards in separate processes: 64-byte cudaIpcMemHandle_t of this buffer,
 * and open all shards' handles (shard_count x 64 bytes, own entry ignored) */
rf_status rf_shard_sync_ipc_handle(rf_volume *vol, void *handle);
rf_status rf_shard_sync_ipc_open(rf_volume *vol, const void *handles);

/* Pre-allocate what a call may otherwise allocate lazily: op records for
 * max_ops ops, the host-keyframe staging ring for width x height keyframes
 * (colour included) and the footprint memo arena.  Connected shards call it
 * before their lockstep phase: growing a buffer synchronises the device,
 * which must not happen while a peer on the same device waits in
 * k_shard_sync (shards emulated in one process). */
rf_status rf_reserve(rf_volume *vol, int32_t width, int32_t height, int32_t max_ops);

/* ---- measurement -------------------------------------------------------- */
rf_status rf_profile_begin(rf_volume *vol);
rf_status rf_profile_end(rf_volume *vol, rf_profile *out);

/* ---- keyframe fusion (keyframe_fusion.py:142-460) ---------------------- */
/* Multiply-add order of the host BLAS behind geometry.transform
 * (p @ R.T + t, src/refusion/geometry.py:101-104): the reference's fused
 * depth depends on it, so it is calibrated on the host and passed in. */
typedef enum rf_blas_order {
    RF_BLAS_PLAIN = 0,    /* (p0 r0 + p1 r1) + p2 r2, no FMA */
    RF_BLAS_FMA_210 = 1,  /* fma(p2, r2, fma(p1, r1, p0 r0)) (OpenBLAS SkylakeX dgemm) */
    RF_BLAS_FMA_012 = 2,  /* fma(p0, r0, fma(p1, r1, p2 r2)) */
    RF_BLAS_FMA_201 = 3   /* fma(p2, r2, fma(p0, r0, p1 r1)) */
} rf_blas_order;

/* depth_sample_weight / discontinuity_mask (keyframe_fusion.py:191-231,
 * :245-246).  flags = RF_DW_MASK: w_map[h][w] = cos(theta)/Z^2 zeroed at
 * discontinuities (fuse_depth's weight map); 0: the unmasked weight;
 * RF_DW_MASK_ONLY: the mask itself as 1.0 / 0.0. */
enum { RF_DW_MASK = 1, RF_DW_MASK_ONLY = 2 };
rf_status rf_depth_weight(const double *depth, int32_t width, int32_t height,
                          double fx, double fy, double cx, double cy,
                          double delta_disc, int32_t flags, double *w_map, void *stream);
/* normal_map (keyframe_fusion.py:142-188): normals[h][w][3], zero at the
 * border and next to invalid depth. */
rf_status rf_normal_map(const double *depth, int32_t width, int32_t height,
                        double fx, double fy, double cx, double cy,
                        double *normals, void *stream);
/* depth_sample_weight(depth, intr, normals) (keyframe_fusion.py:191-208)
 * with caller-supplied normals[h][w][3]. */
rf_status rf_depth_sample_weight_normals(const double *depth, const double *normals,
                                         int32_t width, int32_t height, double fx,
                                         double fy, double cx, double cy, double *w,
                                         void *stream);
/* fuse_depth's warp + np.add.at scatter + Eq. 1 merge (keyframe_fusion.py:
 * 247-276): rel = compose(inverse(kf.pose), frame.pose).  Deterministic:
 * contributions to a keyframe pixel are summed in source-pixel order. */
rf_status rf_fuse_depth(double *kf_depth, double *kf_weight, const double *frame_depth,
                        const double *w_map, int32_t width, int32_t height,
                        double fx, double fy, double cx, double cy,
                        const rf_pose *rel, int32_t blas_order, void *stream);
/* One frame of fuse_depth (keyframe_fusion.py:238-296) in one call: the
 * member's weight map (depth_sample_weight masked by discontinuity_mask,
 * delta_disc) into w_map, its depth copy into depth_copy, the warp +
 * np.add.at scatter + Eq. 1 merge into the keyframe planes (as
 * rf_fuse_depth), and -- frame_color non-null -- the colour prep of
 * rf_color_prep into member_color / blur_weight.  Replaces the reference's
 * per-frame sequence of whole-image numpy passes (:245-296). */
rf_status rf_fuse_frame(double *kf_depth, double *kf_weight, const double *frame_depth,
                        const double *frame_color, int32_t width, int32_t height,
                        double fx, double fy, double cx, double cy, const rf_pose *rel,
                        int32_t blas_order, double delta_disc, const double *gauss_weights,
                        int32_t radius, double gain, double *w_map, double *depth_copy,
                        double *member_color, double *blur_weight, void *stream);
/* unsharp_mask (keyframe_fusion.py:335-346) of an [h][w][channels] image:
 * scipy gaussian_filter (mode 'nearest', gauss_weights[2*radius+1] =
 * _gaussian_kernel1d) per channel, then clip(img + gain*(img - low), 0, 255). */
rf_status rf_unsharp_mask(const double *img, int32_t width, int32_t height, int32_t channels,
                          const double *gauss_weights, int32_t radius, double gain,
                          double *out, void *stream);
/* grayscale (:303-307) of [h][w][3] */
rf_status rf_grayscale(const double *color, int32_t width, int32_t height, double *gray,
                       void *stream);
/* blurriness (:310-332) of a gray [h][w] image; result is a device scalar */
rf_status rf_blurriness(const double *gray, int32_t width, int32_t height,
                        double *blur_weight, void *stream);
/* fuse_depth's colour prep (:278-281): unsharp mask + blurriness of grayscale */
rf_status rf_color_prep(const double *color, int32_t width, int32_t height,
                        const double *gauss_weights, int32_t radius, double gain,
                        double *member_color, double *blur_weight, void *stream);

/* One retained member observation (_MemberObservation, keyframe_fusion.py:87-96). */
typedef struct rf_member_view {
    const double *depth;        /* [h][w] device */
    const double *w_map;        /* [h][w] device */
    const double *color;        /* deblurred [h][w][3] device */
    const double *blur_weight;  /* device scalar */
    rf_pose rel;                /* compose(inverse(member.pose), kf.pose) */
} rf_member_view;

/* fuse_color (keyframe_fusion.py:377-460): per-channel blur-weighted
 * median over any number of members (<= 64: one pass with the samples in
 * registers / local memory; more: global-scratch pass in pixel chunks);
 * color_valid[h][w] is 0/1. */
rf_status rf_fuse_color(const double *kf_depth, const double *kf_weight,
                        int32_t width, int32_t height, double fx, double fy,
                        double cx, double cy, int32_t n_members,
                        const rf_member_view *members, double delta_occl,
                        int32_t blas_order, double *kf_color, uint8_t *color_valid,
                        void *stream);

/* ---- self-tests --------------------------------------------------------- */
/* Compare the kernels' shared-denominator division (Markstein correction)
 * with the IEEE double division on n random operand pairs whose exponents
 * span [-exp_span, exp_span]; *mismatches = differing bit patterns. */
rf_status rf_selftest_division(uint64_t n, uint64_t seed, int32_t exp_span,
                               uint64_t *mismatches);

/* Compare the screened voxel projection (approximate reciprocal + exact
 * fallback near pixel boundaries) with the exact IEEE projection on n
 * random camera points around a width x height image with centre (cx, cy),
 * half of them snapped within a few ulps of a pixel boundary;
 * *mismatches = points whose pixel (or in/out decision) differs. */
rf_status rf_selftest_projection(int32_t width, int32_t height, double cx, double cy,
                                 uint64_t n, uint64_t seed, uint64_t *mismatches);

/* ---- synthetic data (measurement infrastructure, synth.py:46-283) ------ */
typedef struct rf_synth_prim {
    int32_t kind;        /* 0 Sphere (size[0] = radius), 1 BoxSolid, 2 RoomShell */
    int32_t _pad;
    double center[3];
    double size[3];      /* half extents (box / room) */
    double albedo[3];
} rf_synth_prim;

/* Faithful renderer: render_depth / render_color of
 * synth.py:220-267 bit for bit (numpy's evaluation order; the two BLAS
 * products in the host's calibrated order).  Depth noise is drawn on the
 * host by numpy (synth.py:270-283, PCG64 stream); colour shades the noisy
 * depth as make_sequence does. */
typedef struct rf_synth_ref_params {
    double z_max;        /* render_depth z_max (Z_MAX_DEFAULT 10.0) */
    double tol;          /* SPHERE_TRACE_TOL */
    double ambient, diffuse;   /* AMBIENT, DIFFUSE */
    double neg_light[3]; /* -light_dir (render_color's normal @ (-light_dir)) */
    double normal_eps;   /* _NORMAL_EPS */
    int32_t steps;       /* SPHERE_TRACE_STEPS */
    int32_t gemm_order;  /* rf_blas_order of (n,3) @ (3,3) on the host */
    int32_t gemv_order;  /* rf_blas_order of (n,3) @ (3,) on the host */
    int32_t _pad;
} rf_synth_ref_params;

typedef struct rf_synth_gauss {
    double w[64];        /* w[0] centre, w[j] weight at offset j (symmetric) */
    int32_t r;           /* radius (<= 63) */
    int32_t _pad;
} rf_synth_gauss;

/* render_depth (synth.py:220-250): z-depth [h][w] on the device */
rf_status rf_synth_depth(const rf_synth_prim *prims_dev, int32_t n_prims,
                         const rf_pose *pose, double fx, double fy, double cx,
                         double cy, int32_t width, int32_t height,
                         const rf_synth_ref_params *params, double *depth_dev,
                         void *stream);
/* render_color (synth.py:253-267) of a (noisy) depth map: colour [h][w][3] */
rf_status rf_synth_color(const rf_synth_prim *prims_dev, int32_t n_prims,
                         const rf_pose *pose, double fx, double fy, double cx,
                         double cy, int32_t width, int32_t height,
                         const rf_synth_ref_params *params, const double *depth_dev,
                         double *color_dev, void *stream);
/* gaussian_filter(color, sigma=(s, s, 0)) in place (mode 'reflect',
 * synth.py:353-355); tmp_dev: h*w*3 doubles of scratch */
rf_status rf_synth_blur(double *color_dev, double *tmp_dev, int32_t width,
                        int32_t height, const rf_synth_gauss *g, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* REFUSION_B200_H */
