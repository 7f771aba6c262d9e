/*
 * mdrt.h -- C ABI of the B200 multi-depth-camera renderer (libmdrt.so).
 *
 * The reference renderer (`multidepth`, /root/reference/pkg/src/multidepth) is a
 * Python package whose operator/plugin seam is the backend registry
 * `kernels.get_render_fn(name) -> render_batch(...)` (kernels/__init__.py:53-60).
 * Every entry point below replaces one piece of that path; the cited
 * file:line is the reference interface it stands in for. All pointers are
 * plain host or device pointers with explicit sizes; there are no torch
 * types in any signature. Functions return 0 on success and a negative
 * MDRT_E* code on failure; mdrt_last_error() then holds a message
 * (thread-local). Python raises ValueError for MDRT_EINVAL and RuntimeError
 * otherwise, matching the reference's error behaviour (kernels/__init__.py:38-50,
 * scene.py:228-250).
 *
 * Units/conventions follow the reference exactly: quaternions are (w,x,y,z);
 * camera frame +z forward, +x right, +y down (camera.py:3-7); pixel centres at
 * +0.5 (camera.py:83-84); output is Euclidean range in metres; a miss reads
 * exactly float32(d_max) (scene.py:336-338).
 */
#ifndef MDRT_H
#define MDRT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MDRT_ABI_VERSION 2   /* 2: link_states/link_map in mdrt_step_args, peer/bvh/query/depth_to_u8 calls */

#define MDRT_OK 0
#define MDRT_EINVAL -1   /* bad argument (shape/range/state)            */
#define MDRT_ECUDA -2    /* CUDA runtime error (no device, launch, OOM) */
#define MDRT_ESTATE -3   /* call out of order (e.g. render before commit) */

/* flags for mdrt_step_args.flags */
#define MDRT_EARLY_TERMINATION 0x1 /* bound each query by the best hit so far (numba_backend.py:191) */
#define MDRT_SENSOR 0x2            /* fused noise/dropout/clamp epilogue (sensor.py:55-82)          */
#define MDRT_LATENCY 0x4           /* fused latency ring write + delayed read (sensor.py:103-150)   */
#define MDRT_COUNT 0x8             /* count BVH node visits / triangle tests into `counters`         */
#define MDRT_NO_CULL 0x10          /* disable per-view link culling (debug / A-B parity)            */
#define MDRT_PHASE_PROLOGUE 0x20   /* launch only the per-view prologue (timing); neither phase flag = both */
#define MDRT_PHASE_TRACE 0x40      /* launch only the traversal kernel (uses the last prologue's records)  */
#define MDRT_COUNT_DETAIL 0x80     /* with MDRT_COUNT: counters has 4 slots (+ link node fetches, link traversals) */
#define MDRT_RSM 0x200             /* random side masking of the output (perception.py:169-202)             */
#define MDRT_ROT_XYZW 0x400       /* link_states quaternions are stored x, y, z, w (simulator order)     */
#define MDRT_WIDE_STORES 0x800    /* `out` is remote (peer-mapped) memory: render 8-pixel-wide tiles so each
                                     warp's obs stores cover >= 32 contiguous bytes per image row (NVLink
                                     writes in whole sectors instead of 16 B pieces)                      */
#define MDRT_NO_TILE_ENTRY 0x1000 /* trace the terrain from its root instead of each pixel tile's entry node
                                     (entry_kernel's frustum descent; results are identical). Neither this
                                     nor MDRT_TILE_ENTRY: entries when the terrain has >= 65,536 triangles */
#define MDRT_TILE_ENTRY 0x2000    /* per-tile terrain entry nodes regardless of the terrain size          */
#define MDRT_DEVICE_STATE 0x100    /* step, timestamp, RNG prefix and ring push come from the context's device
                                      state (mdrt_state_set), advanced on the device at the start of the call:
                                      the call is then CUDA-graph capturable and replayable with no host args */

typedef struct mdrt_ctx mdrt_ctx;

/* Per-context statistics (mdrt_get_stats). */
typedef struct {
    int64_t num_bodies;
    int64_t body_triangles;
    int64_t body_nodes;
    int64_t terrain_triangles;
    int64_t terrain_nodes;
    int64_t terrain_depth;       /* max depth of the terrain tree (root = 0)           */
    int64_t body_max_depth;      /* max depth over the link trees                      */
    int64_t node_bytes;          /* device bytes of all BVH node records (64 B each)   */
    int64_t tri_bytes;           /* device bytes of all triangle records (48 B each)   */
    int64_t node_record_size;    /* 64                                                 */
    int64_t tri_record_size;     /* 48                                                 */
} mdrt_stats;

/* One render step. Device pointers unless noted. Shapes use N = num_envs of
 * this call (an env slice), B = bodies, C = cameras, H x W pixels. */
typedef struct {
    int32_t num_envs;          /* N (this slice)                                      */
    int32_t flags;             /* MDRT_* flags                                        */
    int64_t env_offset;        /* global index of env 0 of this slice (RNG counter)   */

    /* body poses: replaces Scene.set_body_poses state (scene.py:235-250) */
    const float *body_pos;     /* (N,B,3)                                             */
    const float *body_rot;     /* (N,B,4) wxyz, any nonzero norm (normalised on device) */

    /* per-(env,cam) randomisation: Scene.set_camera_randomization (scene.py:256-273) */
    const float *cam_off_pos;  /* (N,C,3) or NULL                                     */
    const float *cam_off_rot;  /* (N,C,4) or NULL                                     */
    const float *fov_delta;    /* (N,C) degrees or NULL                               */

    /* seam mode (render_batch, numba_backend.py:222): precomposed camera poses and
     * per-pixel ray grids. When cam_pos != NULL the rig/body composition is skipped. */
    const float *cam_pos;      /* (N,C,3) or NULL                                     */
    const float *cam_rot;      /* (N,C,4) or NULL                                     */
    const float *ray_dirs;     /* (RN,C,H,W,3) camera-frame dirs or NULL (intrinsics) */
    const float *ray_scale;    /* (RN,C,H,W) |dir| or NULL                            */
    int32_t ray_envs;          /* RN: 1 (shared) or N                                 */

    /* sensor model: apply_noise_dropout (sensor.py:55-82) */
    double noise_scale;
    double dropout_p;
    const double *fill;        /* HOST (C,) dropout fill per camera, NULL -> d_max    */
    uint64_t sensor_key;       /* rng.stream_key(seed, "sensor") (rng.py:61-68)       */
    int64_t step;              /* counter `step` of the sensor stream                 */

    /* latency ring: FrameBuffer push + fetch_delayed_batch (sensor.py:103-150) */
    float *ring;               /* (R,N,C,H,W)                                         */
    int32_t ring_slots;        /* R                                                   */
    int32_t write_slot;        /* slot receiving this step's frame                    */
    int32_t ring_count;        /* K frames retained after this push (<= R, <= 32)     */
    const double *ring_times;  /* HOST (K,) timestamps, oldest first (incl. this one) */
    const int32_t *ring_order; /* HOST (K,) slot of each retained frame, oldest first */
    double now;                /* fetch time                                          */
    const double *delays;      /* (N,) per-env delay, device                          */
    int32_t *read_slot;        /* (N,) scratch/out: selected slot per env, device      */

    float *out_clean;          /* (N,C,H,W) clean range depth, or NULL                */
    float *out;                /* (N,C,H,W) final output (sensor/latency applied)     */
    unsigned long long *counters; /* (2,) device [node fetches, triangle tests] or NULL; (4,) with MDRT_COUNT_DETAIL */

    /* random side masking: rsm_apply (perception.py:169-202) applied to `out` */
    const int32_t *rsm_modes;  /* (N,C) mode per view (0 none, 1 small, 2 large), device */
    int32_t rsm_k1, rsm_k2;    /* columns masked per side for modes 1 and 2 (int(f * W))  */
    uint64_t rsm_key;          /* rng.stream_key(seed, "rsm-fill")                        */
    double rsm_fill_low;       /* fill ~ U[fill_low, fill_high[c])                        */
    const double *rsm_fill_high; /* HOST (C,), NULL -> d_max                              */

    /* fused downsample_min (sensor.py:85-100) of the final output */
    float *ds_out;             /* (N,C,H/f,W/f) block minimum, or NULL; `out` may then be NULL */
    int32_t ds_factor;         /* f; H and W must be divisible by f                          */

    /* zero-copy pose source (device-side pose ingestion from a
     * simulator's link-state tensor). When non-NULL it replaces body_pos/body_rot:
     * body b of env e reads the record link_states + (e * env_stride + link_map[b]) *
     * record_stride floats, position at +pos_offset, quaternion at +rot_offset (wxyz,
     * or xyzw with MDRT_ROT_XYZW). */
    const float *link_states;
    int64_t env_stride;        /* records per env                                        */
    int32_t record_stride;     /* floats per record (e.g. 13: pos, quat, lin vel, ang vel) */
    int32_t pos_offset;
    int32_t rot_offset;
    const int32_t *link_map;   /* (B,) device: record index of each body within its env  */
} mdrt_step_args;

/* ---- library ---------------------------------------------------------- */
int mdrt_abi_version(void);
const char *mdrt_last_error(void);
/* number of visible CUDA devices (0 on a host without a GPU) */
int mdrt_device_count(int32_t *count);

/* ---- context: replaces Scene geometry state (scene.py:159-211) --------- */
int mdrt_create(int32_t device, mdrt_ctx **out);
int mdrt_destroy(mdrt_ctx *ctx);

/* Register a body (link) mesh in its local frame; SAH BVH built once on the
 * host. Replaces Body/build_bvh (scene.py:165-176, bvh.py:68-136). Triangles
 * with area < 1e-12 are expected to be removed by the caller (mesh.py:47-56).
 * Meshes with non-finite vertices, or with more triangles than the 24-entry
 * traversal stack allows (leaf_max * 2^23: 33.5M at leaves of <= 4, 67M for
 * meshes of >= 500k triangles, whose leaves hold <= 8), return MDRT_EINVAL;
 * so does mdrt_set_terrain. */
int mdrt_add_body(mdrt_ctx *ctx, const double *verts, int64_t nv, const int64_t *faces,
                  int64_t nf, int32_t *body_id);
/* Set the static world-frame terrain mesh (scene.py:191-196). */
int mdrt_set_terrain(mdrt_ctx *ctx, const double *verts, int64_t nv, const int64_t *faces,
                     int64_t nf);
/* Camera rig: CameraModel (camera.py:20-65) x C. parent[c] = body index or -1
 * (mount is a world pose, scene.py:286-287). mount_rot (C,4) wxyz. HOST arrays. */
int mdrt_set_cameras(mdrt_ctx *ctx, int32_t C, int32_t W, int32_t H, const double *hfov_deg,
                     const double *vfov_deg, const double *d_max, const int32_t *parent,
                     const double *mount_pos, const double *mount_rot);
/* Upload all geometry to the device; geometry is immutable afterwards
 * (test_render.py:252-265 "BVHs never rebuilt"). */
int mdrt_commit(mdrt_ctx *ctx);
int mdrt_get_stats(mdrt_ctx *ctx, mdrt_stats *out);

/* ---- per step ----------------------------------------------------------
 * Replaces render() (scene.py:332-348) -> render_batch (numba_backend.py:222-234)
 * and, with MDRT_SENSOR / MDRT_LATENCY, the sensor stage apply_noise_dropout
 * (sensor.py:55-82) and FrameBuffer push/fetch_delayed_batch (sensor.py:122-150),
 * fused into one traversal kernel. `stream` is a cudaStream_t (NULL = default). */
int mdrt_render(mdrt_ctx *ctx, const mdrt_step_args *args, void *stream);

/* Stream ordering of one context. All renders of a context share its per-step
 * scratch (view/link records, tile counters, device step state). Outside CUDA
 * graph capture mdrt_render orders itself: a call on a stream other than the
 * previous call's first waits for that call's completion (cudaStreamWaitEvent).
 * A captured graph runs outside mdrt_render, so its replays are bracketed by
 * mdrt_order_begin (wait for the context's last work) and mdrt_order_end (record
 * the replay as the context's last work) on the replay stream. */
int mdrt_order_begin(mdrt_ctx *ctx, void *stream);
int mdrt_order_end(mdrt_ctx *ctx, void *stream);

/* Device step state for graph replay (MDRT_DEVICE_STATE). Each mdrt_render with
 * the flag first advances it on the device: k = next_step, now = t0 + k*dt,
 * sensor stream prefix from (key, k), and (ring_slots > 0) a FrameBuffer push of
 * `now` into the ring (sensor.py:122-131). times/order: HOST (count,) current
 * ring content, oldest first. Also reserves per-step scratch for num_envs so
 * that later calls allocate nothing (capture-safe). Synchronous. */
int mdrt_state_set(mdrt_ctx *ctx, int32_t num_envs, uint64_t sensor_key, uint64_t rsm_key, double t0,
                   double dt, int64_t next_step, int32_t ring_slots, const double *times,
                   const int32_t *order, int32_t count);
/* Read back the device step state (next_step, now, write_slot, count, times, order). */
int mdrt_state_get(mdrt_ctx *ctx, int64_t *next_step, double *now, int32_t *write_slot, int32_t *count,
                   double *times, int32_t *order);

/* Standalone sensor epilogue on an existing (N,C,H,W) depth tensor
 * (apply_noise_dropout, sensor.py:55-82). d_max/fill: HOST (C,). */
int mdrt_noise_dropout(const float *depth, float *out, int32_t N, int32_t C, int32_t H,
                       int32_t W, int64_t env_offset, const double *d_max, const double *fill,
                       double noise_scale, double dropout_p, uint64_t key, int64_t step,
                       void *stream);

/* FrameBuffer.fetch_delayed_batch gather (sensor.py:141-150): out[e] = frames[slot[e]][e].
 * frames: R device pointers packed in a HOST array; slot: (N,) device. */
int mdrt_gather_delayed(const float *const *frames, int32_t R, const int32_t *slot, float *out,
                        int64_t N, int64_t frame_elems_per_env, void *stream);

/* Per-env slot selection on device (sensor.py:138-139): slot[e] = order[max(bisect_right(
 * times, now - delays[e]) - 1, 0)]. times/order: HOST (K,), K <= 32. */
int mdrt_select_slots(const double *times, const int32_t *order, int32_t K, double now,
                      const double *delays, int32_t *slot, int64_t N, void *stream);

/* rsm_apply (perception.py:169-202) on an existing (N,C,H,W) tensor: side bands of
 * k[mode] columns get U[fill_low, fill_high[c]) from the "rsm-fill" stream keyed
 * (step, env_offset + e, c, row, col); other pixels are copied. modes: (N,C)
 * device; k: HOST (3,); fill_high: HOST (C,). */
int mdrt_rsm_apply(const float *in, float *out, int32_t N, int32_t C, int32_t H, int32_t W,
                   const int32_t *modes, const int32_t *k, uint64_t key, int64_t step, int64_t env_offset,
                   double fill_low, const double *fill_high, void *stream);

/* downsample_min (sensor.py:85-100): block minimum over trailing (H,W). */
int mdrt_downsample_min(const float *in, float *out, int64_t planes, int32_t H, int32_t W,
                        int32_t factor, void *stream);

/* build_bvh (bvh.py:68-136) for one mesh, host only: the same SAH build and
 * packed records the renderer uploads (64 B nodes: both children's fp32 boxes
 * + refs, >= 0 inner index, < 0 ~((first << 3) | (count - 1)); 48 B triangles
 * {v0 + face id, e1, e2}), root = node 0. counts = {nodes, triangles, depth}.
 * Output buffers may be NULL (sizes only); nodes needs <= max(nf, 1) records,
 * tris/tri_index nf entries. leaf_max: 1..8, 0 = default (4). */
int mdrt_bvh_build(const double *verts, int64_t nv, const int64_t *faces, int64_t nf, int32_t leaf_max,
                   void *nodes, int64_t node_cap, void *tris, int64_t tri_cap, int64_t *tri_index,
                   int64_t counts[3]);

/* query_bvh (bvh.py:189-217) for n independent rays on the device: closest hit
 * t in (1e-6, t_max] (+inf on miss) and its original face index (-1 on miss)
 * against a packed tree (device copies of mdrt_bvh_build's nodes/tris).
 * origins/dirs: (n, 3) float32 device; t_max may be +inf. */
int mdrt_query_rays(const void *nodes, const void *tris, const float *origins, const float *dirs, int64_t n,
                    float t_max, float *t_out, int32_t *face_out, void *stream);

/* depth_to_u8 (frameio.py depth_to_u8, PGM previews): out[i] =
 * round_half_even(255 * (1 - clip(in[i] / d_max, 0, 1))) in f64. in: 16-byte
 * aligned device float32; out: 4-byte aligned device uint8. */
int mdrt_depth_to_u8(const float *in, uint8_t *out, int64_t n, double d_max, void *stream);

/* Host-only BVH check (no device needed): builds the packed tree for one mesh
 * exactly as mdrt_add_body/mdrt_set_terrain do and verifies its invariants
 * (every triangle in exactly one leaf, child boxes enclose their triangles,
 * depth <= 24, the traversal stack). Fills info = {nodes, triangles, depth, leaves}. Returns
 * MDRT_EINVAL with a message when an invariant fails. */
int mdrt_bvh_check(const double *verts, int64_t nv, const int64_t *faces, int64_t nf,
                   int64_t info[4]);

/* Bandwidth probe for roofline denominators: `iters` passes of 32-byte L1-bypassing
 * loads (ld.global.cg, 4 blocks of 256 threads per SM) over a device buffer of `bytes`
 * (L2-resident when bytes << L2 size; bytes must be a multiple of 32); writes one
 * float per block into `sink` (device, >= 4096 floats) so loads are live. */
int mdrt_probe_read(const void *buf, int64_t bytes, int32_t iters, float *sink, void *stream);

/* Fault in a HOST buffer's pages from `threads` threads (one write per 4 KB page,
 * values unchanged). The reference's render() hands its backend a freshly
 * allocated numpy `out` (scene.py:344-347); touching it while the GPU renders
 * takes the first-touch page faults off the critical path of the device->host
 * copy into it (kernels/cuda_backend.py). */
int mdrt_host_touch(void *ptr, int64_t bytes, int32_t threads);
/* memcpy of HOST memory by up to `threads` threads of the same persistent pool, in
 * 4 KB-aligned slices (each page of a fresh `dst` is first touched by one thread). */
int mdrt_host_copy(void *dst, const void *src, int64_t bytes, int32_t threads);

/* Fused frame gather over peer memory (the reference
 * has no multi-GPU path, its closest interface is the caller-allocated `out`
 * of render_batch, numba_backend.py:222-234). The destination rank allocates
 * the full (N_total, C, H, W) observation buffer with mdrt_peer_alloc and
 * publishes the 64-byte CUDA IPC handle; every other rank maps it with
 * mdrt_peer_open and passes `mapped + env_offset*C*H*W` as mdrt_step_args.out,
 * so the render epilogue stores its block straight into the destination GPU
 * over NVLink. Ordering between producers and the consumer is the caller's
 * (a stream-ordered collective barrier). */
#define MDRT_IPC_HANDLE_BYTES 64
int mdrt_peer_alloc(int32_t device, int64_t bytes, void **dptr, uint8_t *handle);
int mdrt_peer_open(int32_t device, const uint8_t *handle, void **dptr);
int mdrt_peer_close(void *dptr);  /* unmap a mapping made by mdrt_peer_open */
int mdrt_peer_free(void *dptr);   /* free a buffer made by mdrt_peer_alloc */

/* Synchronise the context's device (debug/tests). */
int mdrt_sync(mdrt_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* MDRT_H */
