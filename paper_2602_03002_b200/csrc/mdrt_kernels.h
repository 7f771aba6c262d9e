// Kernel parameter blocks and declarations (see mdrt_kernels.cu).
#pragma once

#include <cstdint>

#include "mdrt_device.cuh"

namespace mdrt {

// Device-resident per-step bookkeeping for graph replay (MDRT_DEVICE_STATE):
// advance_kernel produces step k's RNG prefixes, timestamp and latency-ring
// push exactly as the host path would (FrameBuffer._reserve semantics).
constexpr int kTileCounters = 1025;   // <= 1024 SM chunks + the shared pool

struct StepState {
    unsigned long long key;       // rng.stream_key(seed, "sensor")
    unsigned long long hu_step;   // absorb(absorb(key, 0), k)
    unsigned long long hn_step;   // absorb(absorb(key, 1), k)
    long long next_step;          // k of the next advance
    double t0, dt, now;           // now = t0 + k * dt
    int32_t ring_slots, ring_count, write_slot, pad;
    double times[32];             // retained timestamps, oldest first
    int32_t order[32];            // their ring slots
    unsigned long long rsm_key;   // rng.stream_key(seed, "rsm-fill")
    unsigned long long hr_step;   // absorb(rsm_key, k)
};

struct PrologueParams {
    int32_t N, C, B, W, H;
    int64_t env_offset;
    const CamRig* rigs;
    const BodyInfo* bodies;
    const float* body_pos;
    const float* body_rot;
    const float* link_states;   // strided simulator link states (replaces body_pos/rot) or NULL
    int64_t env_stride;
    int32_t record_stride, pos_offset, rot_offset, rot_xyzw;
    const int32_t* link_map;
    const float* off_pos;
    const float* off_rot;
    const float* fov_delta;
    const float* cam_pos;   // seam mode
    const float* cam_rot;
    int32_t grid_mode;      // per-pixel ray grids given: no image-space cull
    int32_t no_cull;
    unsigned long long hu_step, hn_step;
    // latency selection
    int32_t latency;
    int32_t ring_count;
    int32_t write_slot;
    double now;
    const double* delays;
    double ring_times[32];
    int32_t ring_order[32];
    int32_t* read_slot_out;
    ViewRec* views;
    LinkRec* links;
    int2* rects;                  // (N*C, B) packed pixel rects of the compacted links (x0|x1<<16, y0|y1<<16)
    unsigned int* reset_counter;  // render kernel's tile counters, zeroed here (prologue runs first)
    int32_t reset_count;          // number of counters to zero
    const StepState* state;       // non-null: step/ring/RNG fields come from device state
    // random side masking (perception.py:169-202)
    const int32_t* rsm_modes;     // (N, C) mode per view or NULL
    int32_t rsm_k[3];             // columns per side for modes 0, 1, 2
    unsigned long long hr_step;   // absorb(rsm key, step)
};

// Per-tile terrain entry nodes (entry_kernel): the deepest terrain-BVH node whose
// sibling subtrees all lie outside the pixel tile's view pyramid.
struct EntryParams {
    const ViewRec* views;
    const float4* nodes;          // packed BVH records (terrain tree at root)
    int32_t root;
    int32_t n_nodes;              // node record count (bounds of the MDRT_CHECKS build)
    int32_t W, H, tile_w, tile_h, tiles_x, tiles_per_view;
    int64_t views_count;          // N * C
    int32_t* out;                 // (N*C, tiles_per_view) entry refs
};

struct RenderParams {
    int32_t N, C, B, W, H;
    int32_t tile_w;               // tile shape: tile_w x (32 / tile_w) pixels (4 or 8)
    int32_t tiles_x, tiles_per_view;
    uint32_t m_tiles_x, m_tiles_per_view, m_C;   // fast_div multipliers floor((2^32-1)/d)
    uint32_t row_tiles, m_row_tiles;             // tiles in one tile row of all views (N * C * tiles_x)
    int32_t row_order;            // tile index order: 1 = tile-row-major over all views, 0 = view-major
    uint32_t order_d1, order_m1;  // first divisor of the tile decode (row_tiles or tiles_per_view) + multiplier
    int32_t early_termination;
    int32_t terrain_root;
    const int32_t* tile_entry;    // per-tile terrain entry refs from the prologue, or NULL (root)
    const float4* nodes;
    const float4* tris;
    int32_t n_nodes, n_tris;      // record counts (bounds of the MDRT_CHECKS build)
    cudaTextureObject_t tri_tex;  // texture object over `tris` (float4 texels): the traversal reads triangles here
    const ViewRec* views;
    const LinkRec* links;
    const int2* rects;
    const float* ray_dirs;
    const float* ray_scale;
    int32_t ray_envs;
    int32_t sensor;
    double noise_scale, dropout_p;
    unsigned long long drop_k;    // drop_threshold(dropout_p)
    double fill[64];
    double dmax64[64];
    float* ring;
    int32_t write_slot;
    int32_t ring_slots;           // frames in `ring` (bounds of the MDRT_CHECKS build)
    int64_t frame;                // N * C * H * W (pixels of one frame)
    float* out_clean;
    float* out;
    unsigned long long* counters;
    unsigned int* tile_counter;   // persistent-warp work counters (zeroed per launch): one per
                                  // SM chunk, then the shared pool (kTileCounters entries)
    int32_t chunks;               // SM-local chunks (0: one shared counter only)
    uint32_t local_tiles;         // tiles [0, local_tiles) are split into `chunks` chunks
    int32_t count_detail;         // counters has 4 slots: + link node fetches, link traversals
    const StepState* state;       // non-null: ring write slot comes from device state
    unsigned int* ds_out;         // (N, C, H/f, W/f) block-min of the observation (float bits) or NULL
    int32_t ds_factor, ds_w, ds_h;
    int32_t rsm;                  // apply side masking to the observation
    double rsm_low;
    double rsm_high[64];
    unsigned long long cmix[512];  // counter_mix(v) for v < 512 (rows and columns of the RNG counters)
};

struct NoiseParams {
    const float* in;
    float* out;
    int32_t N, C, H, W;
    int64_t env_offset;
    unsigned long long hu_step, hn_step;
    double noise_scale, dropout_p;
    unsigned long long drop_k;    // drop_threshold(dropout_p)
    double fill[64];
    double dmax[64];
};

struct RsmParams {
    const float* in;
    float* out;
    const int32_t* modes;
    int32_t N, C, H, W;
    int64_t env_offset;
    int32_t k[3];
    unsigned long long hr_step;
    double low;
    double high[64];
};

struct GatherParams {
    const float* frames[32];
    const int32_t* slot;
    float* out;
    int64_t N, per_env;
};

struct SelectParams {
    double times[32];
    int32_t order[32];
    int32_t K;
    double now;
    const double* delays;
    int32_t* slot;
    int64_t N;
};

struct DownsampleParams {
    const float* in;
    float* out;
    int64_t planes;
    int32_t H, W, f;
};

// Host-side launchers (defined next to the kernels so templates instantiate there).
void launch_prologue(const PrologueParams& p, int64_t views, cudaStream_t s);
void launch_entry(const EntryParams& p, cudaStream_t s);
// geometry_bytes: BVH node + triangle bytes; above the L2 size the tiles are
// scheduled SM-locally (render_kernel) so node reuse comes from L1.
// query_bvh (bvh.py:189-217): closest hit + face of independent rays against one tree
struct QueryParams {
    const float4* nodes;
    const float4* tris;
    int32_t n_nodes, n_tris;
    int32_t root;
    const float* origins;   // (n, 3)
    const float* dirs;      // (n, 3)
    int64_t n;
    float t_max;
    float* t_out;           // (n,) +inf on miss
    int32_t* face_out;      // (n,) -1 on miss
};
void launch_query(const QueryParams& p, cudaStream_t s);

int render_tile_width(int W);   // tile shape the render kernel uses for W-pixel-wide images
void launch_render(const RenderParams& p, int64_t warps, bool count, int64_t geometry_bytes, cudaStream_t s);
void launch_noise(const NoiseParams& p, int64_t total, cudaStream_t s);
void launch_gather(const GatherParams& p, int64_t total, cudaStream_t s);
void launch_select(const SelectParams& p, int64_t n, cudaStream_t s);
void launch_downsample(const DownsampleParams& p, int64_t total, cudaStream_t s);
void launch_depth_u8(const float* in, uint8_t* out, int64_t n, double dmax, cudaStream_t s);
void launch_probe_read(const float4* buf, int64_t n16, int iters, float* sink, cudaStream_t s);
void launch_advance(StepState* st, cudaStream_t s);
void launch_rsm(const RsmParams& p, int64_t total, cudaStream_t s);

}  // namespace mdrt
