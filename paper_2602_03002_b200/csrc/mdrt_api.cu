// C ABI of libmdrt.so (declared in include/mdrt.h).
//
// Host-side ownership mirrors the reference Scene (scene.py:150-211): geometry
// is registered, built once (SAH BVH per mesh, bvh_build.cpp) and committed to
// the device; afterwards only per-step pose/camera/sensor data flows in.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <exception>
#include <limits>
#include <new>
#include <stdexcept>
#include <string>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/mdrt.h"
#include "bvh_build.h"
#include "mdrt_kernels.h"

using namespace mdrt;

namespace {

thread_local std::string g_err;

struct ArgError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct StateError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define CK(expr)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (expr);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            throw CudaError(std::string(#expr) + ": " + cudaGetErrorName(e_) + " (" +             \
                            cudaGetErrorString(e_) + ")");                                         \
    } while (0)

template <class F>
int guarded(F&& f) {
    try {
        f();
        return MDRT_OK;
    } catch (const ArgError& e) {
        g_err = e.what();
        return MDRT_EINVAL;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return MDRT_EINVAL;
    } catch (const StateError& e) {
        g_err = e.what();
        return MDRT_ESTATE;
    } catch (const CudaError& e) {
        g_err = e.what();
        return MDRT_ECUDA;
    } catch (const std::bad_alloc&) {
        g_err = "host out of memory";
        return MDRT_ECUDA;
    } catch (const std::exception& e) {
        g_err = e.what();
        return MDRT_ECUDA;
    }
}

void need(bool ok, const char* msg) {
    if (!ok) throw ArgError(msg);
}

template <class T>
struct DevBuf {
    T* ptr = nullptr;
    size_t cap = 0;  // elements
    void reserve(size_t n) {
        if (n <= cap) return;
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        cap = 0;
        CK(cudaMalloc(&ptr, n * sizeof(T)));
        cap = n;
    }
    void release() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        cap = 0;
    }
};

// Persistent host worker pool for the host-side helpers (mdrt_host_touch/copy):
// spawning threads per call costs more than the work on 25-100 MB buffers.
class HostPool {
   public:
    template <class F>
    void run(int n, F&& f) {
        std::lock_guard<std::mutex> call(call_mu_);   // one parallel region at a time
        n = std::max(1, std::min(n, kMaxWorkers + 1));
        ensure(n - 1);
        std::function<void(int)> job(f);
        {
            std::lock_guard<std::mutex> lk(mu_);
            job_ = &job;
            active_ = n - 1;
            pending_ = n - 1;
            ++gen_;
        }
        cv_.notify_all();
        job(0);
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return pending_ == 0; });
        job_ = nullptr;
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }

   private:
    static constexpr int kMaxWorkers = 63;
    void ensure(int k) {
        while (static_cast<int>(workers_.size()) < k) {
            const int id = static_cast<int>(workers_.size()) + 1;
            workers_.emplace_back([this, id] { loop(id); });
        }
    }
    void loop(int id) {
        uint64_t seen = 0;
        while (true) {
            std::function<void(int)>* job;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                if (id > active_) continue;       // not needed for this region
                job = job_;
            }
            (*job)(id);
            {
                std::lock_guard<std::mutex> lk(mu_);
                if (--pending_ == 0) done_cv_.notify_one();
            }
        }
    }
    std::mutex call_mu_, mu_;
    std::condition_variable cv_, done_cv_;
    std::vector<std::thread> workers_;
    std::function<void(int)>* job_ = nullptr;
    int active_ = 0, pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

HostPool& host_pool() {
    static HostPool pool;
    return pool;
}

}  // namespace

struct mdrt_ctx {
    int device = 0;
    std::vector<PackedTree> bodies;
    PackedTree terrain;
    bool has_terrain = false;
    int32_t node_count = 0, tri_count = 0;   // records uploaded at the last commit
    // cameras
    int32_t C = 0, W = 0, H = 0;
    std::vector<CamRig> rigs;
    bool committed = false;
    // device geometry
    DevBuf<PackedNode> nodes;
    DevBuf<PackedTri> tris;
    DevBuf<BodyInfo> body_info;
    DevBuf<CamRig> rig_buf;
    int32_t terrain_root = -1;
    mdrt_stats stats{};
    // per-step scratch
    DevBuf<ViewRec> views;
    DevBuf<LinkRec> links;
    cudaTextureObject_t tri_tex = 0;   // over `tris`, rebuilt when the buffer changes

    void drop_tri_tex() {
        if (tri_tex) cudaDestroyTextureObject(tri_tex);
        tri_tex = 0;
    }
    cudaTextureObject_t triangle_texture() {
        if (!tri_tex) {
            int max_texels = 0;
            CK(cudaDeviceGetAttribute(&max_texels, cudaDevAttrMaxTexture1DLinearWidth, device));
            need(tris.cap * 3 <= static_cast<size_t>(max_texels),
                 "too many triangles for the texture path (3 texels per triangle)");
            cudaResourceDesc rd{};
            rd.resType = cudaResourceTypeLinear;
            rd.res.linear.devPtr = tris.ptr;
            rd.res.linear.desc = cudaCreateChannelDesc<float4>();
            rd.res.linear.sizeInBytes = tris.cap * sizeof(PackedTri);
            cudaTextureDesc td{};
            td.readMode = cudaReadModeElementType;
            CK(cudaCreateTextureObject(&tri_tex, &rd, &td, nullptr));
        }
        return tri_tex;
    }
    DevBuf<int2> rects;
    DevBuf<int32_t> tile_entry;   // per-tile terrain entry refs (prologue -> render kernel)
    int32_t entry_tile_w = 0;     // tile width the last prologue computed entries for (0: none)
    size_t entry_views = 0;       // and its view count (a trace-only call reuses them only if both match)
    DevBuf<unsigned int> tile_counter;
    DevBuf<StepState> state;
    // Cross-stream ordering of the per-step scratch (views, links, rects, tile
    // counters, step state): every call that uses it waits for the previous
    // user's completion event when it runs on a different stream.
    cudaEvent_t done = nullptr;
    cudaStream_t last_stream = nullptr;
    bool has_last = false;

    void use_device() const { CK(cudaSetDevice(device)); }

    // make `s` wait for this context's last recorded work (no-op on the same stream)
    void order_begin(cudaStream_t s) {
        if (has_last && s != last_stream) CK(cudaStreamWaitEvent(s, done, 0));
    }
    void order_end(cudaStream_t s) {
        if (!done) CK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
        CK(cudaEventRecord(done, s));
        last_stream = s;
        has_last = true;
    }
    static bool capturing(cudaStream_t s) {
        cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
        CK(cudaStreamIsCapturing(s, &st));
        return st != cudaStreamCaptureStatusNone;
    }
};

namespace {
int tiles_per_view_for(int W, int H, int tw) { return ((W + tw - 1) / tw) * ((H + 32 / tw - 1) / (32 / tw)); }
int max_tiles_per_view(int W, int H) { return std::max(tiles_per_view_for(W, H, 4), tiles_per_view_for(W, H, 8)); }
}  // namespace

extern "C" {

int mdrt_abi_version(void) { return MDRT_ABI_VERSION; }

const char* mdrt_last_error(void) { return g_err.c_str(); }

int mdrt_device_count(int32_t* count) {
    return guarded([&] {
        need(count != nullptr, "count is NULL");
        int n = 0;
        cudaError_t e = cudaGetDeviceCount(&n);
        if (e != cudaSuccess) {
            (void)cudaGetLastError();
            n = 0;
        }
        *count = n;
    });
}

int mdrt_create(int32_t device, mdrt_ctx** out) {
    return guarded([&] {
        need(out != nullptr, "out is NULL");
        int n = 0;
        CK(cudaGetDeviceCount(&n));
        need(device >= 0 && device < n, "device index out of range");
        auto* ctx = new mdrt_ctx();
        ctx->device = device;
        *out = ctx;
    });
}

int mdrt_destroy(mdrt_ctx* ctx) {
    return guarded([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        ctx->drop_tri_tex();
        ctx->nodes.release();
        ctx->tris.release();
        ctx->body_info.release();
        ctx->rig_buf.release();
        ctx->views.release();
        ctx->links.release();
        ctx->rects.release();
        ctx->tile_entry.release();
        ctx->tile_counter.release();
        ctx->state.release();
        if (ctx->done) cudaEventDestroy(ctx->done);
        delete ctx;
    });
}

int mdrt_add_body(mdrt_ctx* ctx, const double* verts, int64_t nv, const int64_t* faces, int64_t nf,
                  int32_t* body_id) {
    return guarded([&] {
        need(ctx != nullptr, "ctx is NULL");
        if (ctx->committed) throw StateError("geometry is immutable after mdrt_commit");
        need(verts && faces && nv > 0, "body mesh arrays are empty");
        need(nf > 0, "body has no triangles");
        ctx->bodies.push_back(build_tree(verts, nv, faces, nf));
        if (body_id) *body_id = static_cast<int32_t>(ctx->bodies.size() - 1);
    });
}

int mdrt_set_terrain(mdrt_ctx* ctx, const double* verts, int64_t nv, const int64_t* faces, int64_t nf) {
    return guarded([&] {
        need(ctx != nullptr, "ctx is NULL");
        if (ctx->committed) throw StateError("geometry is immutable after mdrt_commit");
        need(verts && faces && nv > 0, "terrain mesh arrays are empty");
        need(nf > 0, "terrain mesh has no triangles");
        ctx->terrain = build_tree(verts, nv, faces, nf);
        ctx->has_terrain = true;
    });
}

int mdrt_set_cameras(mdrt_ctx* ctx, int32_t C, int32_t W, int32_t H, const double* hfov_deg,
                     const double* vfov_deg, const double* d_max, const int32_t* parent,
                     const double* mount_pos, const double* mount_rot) {
    return guarded([&] {
        need(ctx != nullptr, "ctx is NULL");
        if (ctx->committed) throw StateError("cameras are immutable after mdrt_commit");
        need(C >= 1 && C <= 64, "camera count must be in [1, 64]");
        need(W >= 1 && H >= 1 && W <= 32767 && H <= 32767, "bad image size");
        need(hfov_deg && vfov_deg && d_max && parent && mount_pos && mount_rot, "NULL camera array");
        ctx->C = C;
        ctx->W = W;
        ctx->H = H;
        ctx->rigs.assign(C, CamRig{});
        for (int c = 0; c < C; ++c) {
            CamRig& r = ctx->rigs[c];
            need(hfov_deg[c] > 0 && hfov_deg[c] < 180 && vfov_deg[c] > 0 && vfov_deg[c] < 180,
                 "fov must be in (0, 180) degrees");
            need(d_max[c] > 0, "d_max must be positive");
            for (int a = 0; a < 3; ++a) r.mount_pos[a] = mount_pos[c * 3 + a];
            for (int a = 0; a < 4; ++a) r.mount_rot[a] = mount_rot[c * 4 + a];
            r.hfov_deg = hfov_deg[c];
            r.vfov_deg = vfov_deg[c];
            r.d_max = d_max[c];
            r.parent = parent[c];
        }
    });
}

int mdrt_commit(mdrt_ctx* ctx) {
    return guarded([&] {
        need(ctx != nullptr, "ctx is NULL");
        if (ctx->committed) throw StateError("already committed");
        if (ctx->C < 1) throw StateError("mdrt_set_cameras must precede mdrt_commit");
        const int B = static_cast<int>(ctx->bodies.size());
        for (int c = 0; c < ctx->C; ++c)
            need(ctx->rigs[c].parent >= -1 && ctx->rigs[c].parent < B, "camera parent_body out of range");
        ctx->use_device();
        // concatenate: terrain first, then bodies
        std::vector<PackedNode> nodes;
        std::vector<PackedTri> tris;
        std::vector<BodyInfo> infos;
        mdrt_stats st{};
        auto append = [&](PackedTree& t) -> int32_t {
            const int32_t noff = static_cast<int32_t>(nodes.size());
            const int32_t toff = static_cast<int32_t>(tris.size());
            if (static_cast<int64_t>(tris.size()) + static_cast<int64_t>(t.tris.size()) >= (int64_t(1) << 27))
                throw ArgError("too many triangles (limit 2^27)");
            offset_tree(t, noff, toff);
            nodes.insert(nodes.end(), t.nodes.begin(), t.nodes.end());
            tris.insert(tris.end(), t.tris.begin(), t.tris.end());
            offset_tree(t, -noff, -toff);  // keep the host copy relative
            return noff;
        };
        if (ctx->has_terrain) {
            ctx->terrain_root = append(ctx->terrain);
            st.terrain_nodes = static_cast<int64_t>(ctx->terrain.nodes.size());
            st.terrain_triangles = static_cast<int64_t>(ctx->terrain.tris.size());
            st.terrain_depth = ctx->terrain.depth;
        }
        for (auto& b : ctx->bodies) {
            BodyInfo bi{};
            bi.root = append(b);
            bi.cx = static_cast<float>(b.center[0]);
            bi.cy = static_cast<float>(b.center[1]);
            bi.cz = static_cast<float>(b.center[2]);
            bi.r = static_cast<float>(b.radius * (1.0 + 1e-6)) + 1e-5f;
            // padded half extents of the link AABB around the sphere centre
            bi.hx = static_cast<float>(0.5 * (b.box_hi[0] - b.box_lo[0]) * (1.0 + 1e-5) + 1e-4);
            bi.hy = static_cast<float>(0.5 * (b.box_hi[1] - b.box_lo[1]) * (1.0 + 1e-5) + 1e-4);
            bi.hz = static_cast<float>(0.5 * (b.box_hi[2] - b.box_lo[2]) * (1.0 + 1e-5) + 1e-4);
            infos.push_back(bi);
            st.body_nodes += static_cast<int64_t>(b.nodes.size());
            st.body_triangles += static_cast<int64_t>(b.tris.size());
            st.body_max_depth = std::max<int64_t>(st.body_max_depth, b.depth);
        }
        st.num_bodies = B;
        st.node_record_size = sizeof(PackedNode);
        st.tri_record_size = sizeof(PackedTri);
        st.node_bytes = static_cast<int64_t>(nodes.size() * sizeof(PackedNode));
        st.tri_bytes = static_cast<int64_t>(tris.size() * sizeof(PackedTri));
        if (nodes.empty()) nodes.push_back(PackedNode{});
        if (tris.empty()) tris.push_back(PackedTri{});
        if (infos.empty()) infos.push_back(BodyInfo{});
        ctx->drop_tri_tex();
        ctx->nodes.reserve(nodes.size());
        ctx->tris.reserve(tris.size());
        ctx->node_count = static_cast<int32_t>(nodes.size());
        ctx->tri_count = static_cast<int32_t>(tris.size());
        ctx->body_info.reserve(infos.size());
        ctx->rig_buf.reserve(ctx->rigs.size());
        CK(cudaMemcpy(ctx->nodes.ptr, nodes.data(), nodes.size() * sizeof(PackedNode), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->tris.ptr, tris.data(), tris.size() * sizeof(PackedTri), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->body_info.ptr, infos.data(), infos.size() * sizeof(BodyInfo), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->rig_buf.ptr, ctx->rigs.data(), ctx->rigs.size() * sizeof(CamRig),
                      cudaMemcpyHostToDevice));
        ctx->stats = st;
        ctx->committed = true;
    });
}

int mdrt_get_stats(mdrt_ctx* ctx, mdrt_stats* out) {
    return guarded([&] {
        need(ctx && out, "NULL argument");
        if (!ctx->committed) throw StateError("mdrt_commit first");
        *out = ctx->stats;
    });
}

int mdrt_render(mdrt_ctx* ctx, const mdrt_step_args* a, void* stream) {
    return guarded([&] {
        need(ctx && a, "NULL argument");
        if (!ctx->committed) throw StateError("mdrt_commit must precede mdrt_render");
        const int32_t N = a->num_envs, C = ctx->C, B = static_cast<int32_t>(ctx->bodies.size());
        need(N >= 1, "num_envs must be >= 1");
        need(a->out != nullptr || a->ds_out != nullptr, "out is NULL");
        if (a->ds_out) {
            need(a->ds_factor >= 1 && ctx->H % a->ds_factor == 0 && ctx->W % a->ds_factor == 0,
                 "resolution not divisible by downsample factor");
        }
        need(static_cast<int64_t>(N) * C * ctx->H * ctx->W < (int64_t(1) << 31),
             "num_envs * cameras * H * W must be below 2^31 pixels per step (split the batch)");
        const bool seam = a->cam_pos != nullptr;
        need(!seam || a->cam_rot != nullptr, "cam_rot is NULL while cam_pos is set");
        need(B == 0 || (a->body_pos && a->body_rot) || a->link_states, "body poses are NULL");
        if (a->link_states) {
            need(a->link_map != nullptr, "link_map is NULL while link_states is set");
            need(a->record_stride >= 7 && a->env_stride >= 1, "bad link_states strides");
            need(a->pos_offset >= 0 && a->pos_offset + 3 <= a->record_stride && a->rot_offset >= 0 &&
                     a->rot_offset + 4 <= a->record_stride,
                 "link_states offsets outside the record");
        }
        need(!(a->cam_off_pos || a->cam_off_rot) || (a->cam_off_pos && a->cam_off_rot),
             "cam_off_pos and cam_off_rot must be given together");
        need(!a->ray_dirs || a->ray_scale, "ray_scale is NULL while ray_dirs is set");
        need(!a->ray_dirs || a->ray_envs == 1 || a->ray_envs == N, "ray_envs must be 1 or num_envs");
        const bool sensor = (a->flags & MDRT_SENSOR) != 0;
        const bool latency = (a->flags & MDRT_LATENCY) != 0;
        if (sensor) {
            need(a->noise_scale >= 0, "noise_scale must be >= 0");
            need(a->dropout_p >= 0 && a->dropout_p < 1, "dropout_p must be in [0, 1)");
        }
        const bool dstate = (a->flags & MDRT_DEVICE_STATE) != 0;
        if (dstate && !ctx->state.ptr) throw StateError("MDRT_DEVICE_STATE needs mdrt_state_set first");
        if (latency) {
            need(a->ring && a->ring_slots >= 1 && a->ring_slots <= 32, "ring must have 1..32 slots");
            need(a->delays, "delays is NULL");
            if (!dstate) {
                need(a->write_slot >= 0 && a->write_slot < a->ring_slots, "write_slot out of range");
                need(a->ring_count >= 1 && a->ring_count <= a->ring_slots, "ring_count out of range");
                need(a->ring_times && a->ring_order, "latency arrays are NULL");
            }
        }
        need(!(a->flags & MDRT_COUNT) || a->counters, "counters is NULL with MDRT_COUNT");
        ctx->use_device();
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        // outside graph capture the context orders its own scratch across streams;
        // a captured graph's replays are ordered by mdrt_order_begin/end around them
        const bool ordered = !mdrt_ctx::capturing(s);
        if (ordered) ctx->order_begin(s);
        const size_t nviews = static_cast<size_t>(N) * C;
        ctx->views.reserve(nviews);
        ctx->links.reserve(std::max<size_t>(1, nviews * std::max(B, 1)));
        ctx->rects.reserve(std::max<size_t>(1, nviews * std::max(B, 1)));

        PrologueParams pp{};
        pp.N = N; pp.C = C; pp.B = B; pp.W = ctx->W; pp.H = ctx->H;
        pp.env_offset = a->env_offset;
        pp.rigs = ctx->rig_buf.ptr;
        pp.bodies = ctx->body_info.ptr;
        pp.body_pos = a->body_pos;
        pp.body_rot = a->body_rot;
        pp.link_states = a->link_states;
        pp.env_stride = a->env_stride;
        pp.record_stride = a->record_stride;
        pp.pos_offset = a->pos_offset;
        pp.rot_offset = a->rot_offset;
        pp.rot_xyzw = (a->flags & MDRT_ROT_XYZW) != 0;
        pp.link_map = a->link_map;
        pp.off_pos = seam ? nullptr : a->cam_off_pos;
        pp.off_rot = seam ? nullptr : a->cam_off_rot;
        pp.fov_delta = a->ray_dirs ? nullptr : a->fov_delta;
        pp.cam_pos = a->cam_pos;
        pp.cam_rot = a->cam_rot;
        pp.grid_mode = a->ray_dirs != nullptr;
        pp.no_cull = (a->flags & MDRT_NO_CULL) != 0;
        unsigned long long key = a->sensor_key;
        unsigned long long st = static_cast<unsigned long long>(a->step);
        pp.hu_step = absorb(absorb(key, 0ULL), st);
        pp.hn_step = absorb(absorb(key, 1ULL), st);
        pp.latency = latency;
        pp.state = dstate ? ctx->state.ptr : nullptr;
        const bool rsm = (a->flags & MDRT_RSM) != 0;
        if (rsm) {
            need(a->rsm_modes != nullptr, "rsm_modes is NULL with MDRT_RSM");
            need(a->rsm_k1 >= 0 && a->rsm_k2 >= 0 && 2 * a->rsm_k1 <= ctx->W && 2 * a->rsm_k2 <= ctx->W,
                 "rsm column counts out of range");
            // the fused block minimum (ds_out) orders floats by their bit patterns, which
            // holds for values >= 0 only; every other output value is >= 1e-6 or d_max > 0
            need(!a->ds_out || a->rsm_fill_low >= 0.0, "rsm_fill_low must be >= 0 with ds_out (fused block minimum)");
            pp.rsm_modes = a->rsm_modes;
            pp.rsm_k[0] = 0;
            pp.rsm_k[1] = a->rsm_k1;
            pp.rsm_k[2] = a->rsm_k2;
            pp.hr_step = absorb(a->rsm_key, static_cast<unsigned long long>(a->step));
        }
        if (latency && !dstate) {
            pp.ring_count = a->ring_count;
            pp.write_slot = a->write_slot;
            pp.now = a->now;
            pp.delays = a->delays;
            for (int k = 0; k < a->ring_count; ++k) {
                pp.ring_times[k] = a->ring_times[k];
                need(a->ring_order[k] >= 0 && a->ring_order[k] < a->ring_slots, "ring_order out of range");
                pp.ring_order[k] = a->ring_order[k];
            }
        }
        if (latency) {
            pp.delays = a->delays;
            pp.read_slot_out = a->read_slot;
        }
        pp.views = ctx->views.ptr;
        pp.links = ctx->links.ptr;
        pp.rects = ctx->rects.ptr;
        // tile shape of this call (the prologue computes per-tile terrain entries for it)
        const int tile_w = (a->flags & MDRT_WIDE_STORES) ? 8 : render_tile_width(ctx->W);
        const int tile_h = 32 / tile_w;
        const int tiles_x = (ctx->W + tile_w - 1) / tile_w;
        const int tiles_per_view = tiles_x * ((ctx->H + tile_h - 1) / tile_h);
        // per-tile entry nodes pay for their extra launch on deep terrain trees (config 2
        // +0.9 %, config 5 +2.5 %, paper +1.7 %) but not on small ones (config 3's 8,750
        // triangles: -0.5 %): on by default from 65,536 terrain triangles
        const bool want_entries = (a->flags & MDRT_TILE_ENTRY) ||
                                  (!(a->flags & MDRT_NO_TILE_ENTRY) && ctx->stats.terrain_triangles >= 65536);
        const bool entries = ctx->has_terrain && !pp.grid_mode && want_entries;
        EntryParams ep{};
        if (entries) {
            ctx->tile_entry.reserve(std::max<size_t>(1, nviews * max_tiles_per_view(ctx->W, ctx->H)));
            ep.views = ctx->views.ptr;
            ep.nodes = reinterpret_cast<const float4*>(ctx->nodes.ptr);
            ep.root = ctx->terrain_root;
            ep.n_nodes = ctx->node_count;
            ep.W = ctx->W;
            ep.H = ctx->H;
            ep.tile_w = tile_w;
            ep.tile_h = tile_h;
            ep.tiles_x = tiles_x;
            ep.tiles_per_view = tiles_per_view;
            ep.views_count = static_cast<int64_t>(nviews);
            ep.out = ctx->tile_entry.ptr;
        }
        ctx->tile_counter.reserve(kTileCounters);
        pp.reset_counter = ctx->tile_counter.ptr;
        pp.reset_count = kTileCounters;
        const bool only_pro = (a->flags & MDRT_PHASE_PROLOGUE) && !(a->flags & MDRT_PHASE_TRACE);
        const bool only_trace = (a->flags & MDRT_PHASE_TRACE) && !(a->flags & MDRT_PHASE_PROLOGUE);
        if (dstate && !only_trace) {
            launch_advance(ctx->state.ptr, s);
            CK(cudaGetLastError());
        }
        if (!only_trace) {
            launch_prologue(pp, static_cast<int64_t>(nviews), s);
            CK(cudaGetLastError());
            if (entries) {
                launch_entry(ep, s);
                CK(cudaGetLastError());
            }
            ctx->entry_tile_w = entries ? tile_w : 0;
            ctx->entry_views = nviews;
        }
        // a trace-only call uses the entries of the last prologue only when they were
        // computed for this call's tiles (else: terrain from the root, same result)
        const bool use_entries = entries && (!only_trace || (ctx->entry_tile_w == tile_w && ctx->entry_views == nviews));
        if (only_pro) {
            if (ordered) ctx->order_end(s);
            return;
        }

        RenderParams rp{};
        rp.N = N; rp.C = C; rp.B = B; rp.W = ctx->W; rp.H = ctx->H;
        // remote `out` (fused gather over NVLink): 8-wide tiles, 32 B contiguous per row store
        rp.tile_w = tile_w;
        rp.tiles_x = tiles_x;
        rp.tiles_per_view = tiles_per_view;
        rp.tile_entry = use_entries ? ctx->tile_entry.ptr : nullptr;
        rp.m_tiles_x = static_cast<uint32_t>(0xffffffffu / static_cast<uint32_t>(rp.tiles_x));
        rp.m_tiles_per_view = static_cast<uint32_t>(0xffffffffu / static_cast<uint32_t>(rp.tiles_per_view));
        rp.m_C = static_cast<uint32_t>(0xffffffffu / static_cast<uint32_t>(C));
        rp.row_tiles = static_cast<uint32_t>(N) * static_cast<uint32_t>(C) * static_cast<uint32_t>(rp.tiles_x);
        rp.m_row_tiles = static_cast<uint32_t>(0xffffffffu / rp.row_tiles);
        rp.early_termination = (a->flags & MDRT_EARLY_TERMINATION) != 0;
        rp.terrain_root = ctx->has_terrain ? ctx->terrain_root : -1;
        rp.nodes = reinterpret_cast<const float4*>(ctx->nodes.ptr);
        rp.tris = reinterpret_cast<const float4*>(ctx->tris.ptr);
        rp.n_nodes = ctx->node_count;
        rp.n_tris = ctx->tri_count;
        rp.tri_tex = ctx->triangle_texture();
        for (int i = 0; i < 512; ++i) rp.cmix[i] = counter_mix(static_cast<unsigned long long>(i));
        rp.views = ctx->views.ptr;
        rp.links = ctx->links.ptr;
        rp.rects = ctx->rects.ptr;
        rp.ray_dirs = a->ray_dirs;
        rp.ray_scale = a->ray_scale;
        rp.ray_envs = a->ray_envs;
        rp.sensor = sensor;
        rp.noise_scale = a->noise_scale;
        rp.dropout_p = a->dropout_p;
        rp.drop_k = drop_threshold(a->dropout_p);
        for (int c = 0; c < C; ++c) {
            rp.dmax64[c] = ctx->rigs[c].d_max;
            rp.fill[c] = a->fill ? a->fill[c] : ctx->rigs[c].d_max;
        }
        rp.ring = latency ? a->ring : nullptr;
        rp.write_slot = a->write_slot;
        rp.ring_slots = a->ring_slots;
        rp.frame = static_cast<int64_t>(N) * C * ctx->H * ctx->W;
        rp.out_clean = a->out_clean;
        rp.out = a->out;
        rp.counters = a->counters;
        rp.count_detail = (a->flags & MDRT_COUNT_DETAIL) != 0;
        rp.state = dstate ? ctx->state.ptr : nullptr;
        rp.rsm = rsm;
        rp.ds_out = reinterpret_cast<unsigned int*>(a->ds_out);
        rp.ds_factor = a->ds_factor;
        rp.ds_w = a->ds_out ? ctx->W / a->ds_factor : 0;
        rp.ds_h = a->ds_out ? ctx->H / a->ds_factor : 0;
        if (a->ds_out && !only_pro)   // +inf-like start value for the block minima (0x7f7f7f7f = 3.4e38)
            CK(cudaMemsetAsync(a->ds_out, 0x7f, sizeof(float) * nviews * rp.ds_w * rp.ds_h, s));
        rp.rsm_low = a->rsm_fill_low;
        for (int c = 0; c < C; ++c) rp.rsm_high[c] = a->rsm_fill_high ? a->rsm_fill_high[c] : ctx->rigs[c].d_max;
        ctx->tile_counter.reserve(kTileCounters);
        rp.tile_counter = ctx->tile_counter.ptr;
        const int64_t warps = static_cast<int64_t>(nviews) * rp.tiles_per_view;
        need(warps < (int64_t(1) << 31), "launch too large");
        if (only_trace)   // prologue not run
            CK(cudaMemsetAsync(rp.tile_counter, 0, sizeof(unsigned int) * kTileCounters, s));
        const int64_t geometry_bytes = static_cast<int64_t>(ctx->nodes.cap * sizeof(PackedNode) +
                                                            ctx->tris.cap * sizeof(PackedTri));
        launch_render(rp, warps, (a->flags & MDRT_COUNT) != 0, geometry_bytes, s);
        CK(cudaGetLastError());
        if (ordered) ctx->order_end(s);
    });
}

int mdrt_order_begin(mdrt_ctx* ctx, void* stream) {
    return guarded([&] {
        need(ctx != nullptr, "ctx is NULL");
        ctx->use_device();
        ctx->order_begin(static_cast<cudaStream_t>(stream));
    });
}

int mdrt_order_end(mdrt_ctx* ctx, void* stream) {
    return guarded([&] {
        need(ctx != nullptr, "ctx is NULL");
        ctx->use_device();
        ctx->order_end(static_cast<cudaStream_t>(stream));
    });
}

int mdrt_state_set(mdrt_ctx* ctx, int32_t num_envs, uint64_t sensor_key, uint64_t rsm_key, double t0, double dt,
                   int64_t next_step, int32_t ring_slots, const double* times, const int32_t* order, int32_t count) {
    return guarded([&] {
        need(ctx != nullptr, "ctx is NULL");
        if (!ctx->committed) throw StateError("mdrt_commit first");
        need(num_envs >= 1, "num_envs must be >= 1");
        need(ring_slots >= 0 && ring_slots <= 32, "ring_slots must be in [0, 32]");
        need(count >= 0 && count <= ring_slots, "count out of range");
        need(count == 0 || (times && order), "times/order are NULL");
        ctx->use_device();
        StepState st{};
        st.key = sensor_key;
        st.rsm_key = rsm_key;
        st.next_step = next_step;
        st.t0 = t0;
        st.dt = dt;
        st.ring_slots = ring_slots;
        st.ring_count = count;
        st.write_slot = count > 0 ? order[count - 1] : 0;
        for (int i = 0; i < count; ++i) {
            need(order[i] >= 0 && order[i] < ring_slots, "order entry out of range");
            st.times[i] = times[i];
            st.order[i] = order[i];
        }
        ctx->state.reserve(1);
        const size_t nviews = static_cast<size_t>(num_envs) * ctx->C;
        ctx->views.reserve(nviews);
        ctx->links.reserve(std::max<size_t>(1, nviews * std::max<size_t>(ctx->bodies.size(), 1)));
        ctx->rects.reserve(std::max<size_t>(1, nviews * std::max<size_t>(ctx->bodies.size(), 1)));
        ctx->tile_entry.reserve(std::max<size_t>(1, nviews * max_tiles_per_view(ctx->W, ctx->H)));
        ctx->tile_counter.reserve(kTileCounters);
        CK(cudaMemcpy(ctx->state.ptr, &st, sizeof(st), cudaMemcpyHostToDevice));
    });
}

int mdrt_state_get(mdrt_ctx* ctx, int64_t* next_step, double* now, int32_t* write_slot, int32_t* count,
                   double* times, int32_t* order) {
    return guarded([&] {
        need(ctx != nullptr, "ctx is NULL");
        if (!ctx->state.ptr) throw StateError("no device state (mdrt_state_set)");
        ctx->use_device();
        StepState st{};
        CK(cudaMemcpy(&st, ctx->state.ptr, sizeof(st), cudaMemcpyDeviceToHost));
        if (next_step) *next_step = st.next_step;
        if (now) *now = st.now;
        if (write_slot) *write_slot = st.write_slot;
        if (count) *count = st.ring_count;
        for (int i = 0; i < st.ring_count; ++i) {
            if (times) times[i] = st.times[i];
            if (order) order[i] = st.order[i];
        }
    });
}

int mdrt_noise_dropout(const float* depth, float* out, int32_t N, int32_t C, int32_t H, int32_t W,
                       int64_t env_offset, const double* d_max, const double* fill, double noise_scale,
                       double dropout_p, uint64_t key, int64_t step, void* stream) {
    return guarded([&] {
        need(depth && out && d_max, "NULL argument");
        need(N >= 0 && C >= 1 && C <= 64 && H >= 1 && W >= 1, "bad shape");
        need(noise_scale >= 0, "noise_scale must be >= 0");
        need(dropout_p >= 0 && dropout_p < 1, "dropout_p must be in [0, 1)");
        NoiseParams p{};
        p.in = depth;
        p.out = out;
        p.N = N; p.C = C; p.H = H; p.W = W;
        p.env_offset = env_offset;
        p.hu_step = absorb(absorb(key, 0ULL), static_cast<unsigned long long>(step));
        p.hn_step = absorb(absorb(key, 1ULL), static_cast<unsigned long long>(step));
        p.noise_scale = noise_scale;
        p.dropout_p = dropout_p;
        p.drop_k = drop_threshold(dropout_p);
        for (int c = 0; c < C; ++c) {
            p.dmax[c] = d_max[c];
            p.fill[c] = fill ? fill[c] : d_max[c];
        }
        const int64_t total = static_cast<int64_t>(N) * C * H * W;
        if (total == 0) return;
        launch_noise(p, total, static_cast<cudaStream_t>(stream));
        CK(cudaGetLastError());
    });
}

int mdrt_rsm_apply(const float* in, float* out, int32_t N, int32_t C, int32_t H, int32_t W, const int32_t* modes,
                   const int32_t* k, uint64_t key, int64_t step, int64_t env_offset, double fill_low,
                   const double* fill_high, void* stream) {
    return guarded([&] {
        need(in && out && modes && k && fill_high, "NULL argument");
        need(N >= 0 && C >= 1 && C <= 64 && H >= 1 && W >= 1, "bad shape");
        RsmParams p{};
        p.in = in;
        p.out = out;
        p.modes = modes;
        p.N = N; p.C = C; p.H = H; p.W = W;
        p.env_offset = env_offset;
        for (int i = 0; i < 3; ++i) {
            need(k[i] >= 0 && 2 * k[i] <= W, "mask columns out of range");
            p.k[i] = k[i];
        }
        p.hr_step = absorb(key, static_cast<unsigned long long>(step));
        p.low = fill_low;
        for (int c = 0; c < C; ++c) p.high[c] = fill_high[c];
        const int64_t total = static_cast<int64_t>(N) * C * H * W;
        if (total == 0) return;
        launch_rsm(p, total, static_cast<cudaStream_t>(stream));
        CK(cudaGetLastError());
    });
}

int mdrt_gather_delayed(const float* const* frames, int32_t R, const int32_t* slot, float* out, int64_t N,
                        int64_t per_env, void* stream) {
    return guarded([&] {
        need(frames && slot && out, "NULL argument");
        need(R >= 1 && R <= 32, "1..32 frames");
        GatherParams p{};
        for (int i = 0; i < R; ++i) p.frames[i] = frames[i];
        p.slot = slot;
        p.out = out;
        p.N = N;
        p.per_env = per_env;
        const int64_t total = N * per_env;
        if (total == 0) return;
        launch_gather(p, total, static_cast<cudaStream_t>(stream));
        CK(cudaGetLastError());
    });
}

int mdrt_select_slots(const double* times, const int32_t* order, int32_t K, double now, const double* delays,
                      int32_t* slot, int64_t N, void* stream) {
    return guarded([&] {
        need(times && order && delays && slot, "NULL argument");
        need(K >= 1 && K <= 32, "K must be in [1, 32]");
        SelectParams p{};
        for (int k = 0; k < K; ++k) {
            p.times[k] = times[k];
            p.order[k] = order[k];
        }
        p.K = K;
        p.now = now;
        p.delays = delays;
        p.slot = slot;
        p.N = N;
        if (N == 0) return;
        launch_select(p, N, static_cast<cudaStream_t>(stream));
        CK(cudaGetLastError());
    });
}

int mdrt_downsample_min(const float* in, float* out, int64_t planes, int32_t H, int32_t W, int32_t factor,
                        void* stream) {
    return guarded([&] {
        need(in && out, "NULL argument");
        need(factor >= 1, "factor must be >= 1");
        need(H % factor == 0 && W % factor == 0, "resolution not divisible by downsample factor");
        DownsampleParams p{};
        p.in = in;
        p.out = out;
        p.planes = planes;
        p.H = H;
        p.W = W;
        p.f = factor;
        const int64_t total = planes * (H / factor) * (W / factor);
        if (total == 0) return;
        launch_downsample(p, total, static_cast<cudaStream_t>(stream));
        CK(cudaGetLastError());
    });
}

int mdrt_bvh_build(const double* verts, int64_t nv, const int64_t* faces, int64_t nf, int32_t leaf_max, void* nodes,
                   int64_t node_cap, void* tris, int64_t tri_cap, int64_t* tri_index, int64_t counts[3]) {
    return guarded([&] {
        need(verts && faces && counts, "NULL argument");
        need(leaf_max >= 0 && leaf_max <= 8, "leaf_max must be in [1, 8] (0: default)");
        PackedTree t = build_tree(verts, nv, faces, nf, leaf_max);
        counts[0] = static_cast<int64_t>(t.nodes.size());
        counts[1] = static_cast<int64_t>(t.tris.size());
        counts[2] = t.depth;
        need(!nodes || node_cap >= counts[0], "node buffer too small");
        need(!tris || tri_cap >= counts[1], "triangle buffer too small");
        need(!tri_index || tri_cap >= counts[1], "tri_index buffer too small");
        if (nodes) std::memcpy(nodes, t.nodes.data(), t.nodes.size() * sizeof(PackedNode));
        if (tris) std::memcpy(tris, t.tris.data(), t.tris.size() * sizeof(PackedTri));
        if (tri_index) std::memcpy(tri_index, t.tri_index.data(), t.tri_index.size() * sizeof(int64_t));
    });
}

int mdrt_query_rays(const void* nodes, const void* tris, const float* origins, const float* dirs, int64_t n,
                    float t_max, float* t_out, int32_t* face_out, void* stream) {
    return guarded([&] {
        need(nodes && tris && t_out && face_out, "NULL argument");
        need(n == 0 || (origins && dirs), "NULL rays");
        need(!(t_max < 0.0f), "t_max must be >= 0");
        if (n == 0) return;
        QueryParams q{};
        q.nodes = static_cast<const float4*>(nodes);
        q.tris = static_cast<const float4*>(tris);
        q.n_nodes = q.n_tris = INT32_MAX;   // the ABI passes no record counts
        q.root = 0;
        q.origins = origins;
        q.dirs = dirs;
        q.n = n;
        q.t_max = t_max;
        q.t_out = t_out;
        q.face_out = face_out;
        launch_query(q, static_cast<cudaStream_t>(stream));
        CK(cudaGetLastError());
    });
}

int mdrt_depth_to_u8(const float* in, uint8_t* out, int64_t n, double d_max, void* stream) {
    return guarded([&] {
        need(in && out, "NULL argument");
        need(d_max > 0.0, "d_max must be positive");
        need(reinterpret_cast<uintptr_t>(in) % 16 == 0 && reinterpret_cast<uintptr_t>(out) % 4 == 0,
             "depth_to_u8 needs 16-byte aligned input and 4-byte aligned output");
        if (n <= 0) return;
        launch_depth_u8(in, out, n, d_max, static_cast<cudaStream_t>(stream));
        CK(cudaGetLastError());
    });
}

int mdrt_bvh_check(const double* verts, int64_t nv, const int64_t* faces, int64_t nf, int64_t info[4]) {
    return guarded([&] {
        need(verts && faces && info, "NULL argument");
        PackedTree t = build_tree(verts, nv, faces, nf);
        std::vector<int> seen(t.tris.size(), 0);
        int64_t leaves = 0;
        int maxd = 0;
        // walk: (ref, depth, box of this ref as stored in the parent)
        struct It { int32_t ref; int depth; float lo[3], hi[3]; };
        std::vector<It> st;
        const float inf = std::numeric_limits<float>::infinity();
        st.push_back({0, 0, {-inf, -inf, -inf}, {inf, inf, inf}});
        while (!st.empty()) {
            It it = st.back();
            st.pop_back();
            maxd = std::max(maxd, it.depth);
            if (it.ref >= 0) {
                need(it.ref < static_cast<int32_t>(t.nodes.size()), "node ref out of range");
                const PackedNode& n = t.nodes[it.ref];
                It a{n.ref0, it.depth + 1, {n.c0x0, n.c0y0, n.c0z0}, {n.c0x1, n.c0y1, n.c0z1}};
                It b{n.ref1, it.depth + 1, {n.c1x0, n.c1y0, n.c1z0}, {n.c1x1, n.c1y1, n.c1z1}};
                for (const It* c : {&a, &b}) {
                    if (c->lo[0] > c->hi[0]) continue;  // empty child (single-leaf root)
                    for (int k = 0; k < 3; ++k)
                        need(c->lo[k] >= it.lo[k] && c->hi[k] <= it.hi[k], "child box escapes parent box");
                    st.push_back(*c);
                }
            } else {
                const int32_t v = ~it.ref;
                const int64_t first = v >> 3, cnt = (v & 7) + 1;
                need(cnt <= 8, "leaf larger than the encoding allows");
                need(first + cnt <= static_cast<int64_t>(t.tris.size()), "leaf range out of bounds");
                ++leaves;
                for (int64_t i = first; i < first + cnt; ++i) {
                    need(seen[i] == 0, "triangle referenced by two leaves");
                    seen[i] = 1;
                    const int64_t f = t.tri_index[i];
                    for (int k = 0; k < 3; ++k) {
                        const double* p = verts + faces[f * 3 + k] * 3;
                        for (int a2 = 0; a2 < 3; ++a2)
                            need(p[a2] >= it.lo[a2] && p[a2] <= it.hi[a2], "triangle escapes its leaf box");
                    }
                }
            }
        }
        for (int x : seen) need(x == 1, "triangle not referenced by any leaf");
        need(maxd <= kMaxDepth, "tree deeper than the traversal stack");
        info[0] = static_cast<int64_t>(t.nodes.size());
        info[1] = static_cast<int64_t>(t.tris.size());
        info[2] = maxd;
        info[3] = leaves;
    });
}

int mdrt_probe_read(const void* buf, int64_t bytes, int32_t iters, float* sink, void* stream) {
    return guarded([&] {
        need(buf && sink && bytes >= 16 && iters >= 1, "bad probe arguments");
        launch_probe_read(static_cast<const float4*>(buf), bytes / 16, iters, sink, static_cast<cudaStream_t>(stream));
        CK(cudaGetLastError());
    });
}

int mdrt_host_touch(void* ptr, int64_t bytes, int32_t threads) {
    return guarded([&] {
        need(ptr != nullptr || bytes == 0, "ptr is NULL");
        need(bytes >= 0 && threads >= 1 && threads <= 256, "bad host_touch arguments");
        if (bytes == 0) return;
        // one write per 4 KB page (value unchanged); the pool's threads take contiguous
        // slices, so page faults on different ranges of one mapping proceed in parallel
        constexpr int64_t kPage = 4096;
        volatile char* base = static_cast<volatile char*>(ptr);
        const int64_t pages = (bytes + kPage - 1) / kPage;
        const int n = static_cast<int>(std::min<int64_t>(threads, std::max<int64_t>(1, pages / 64)));
        host_pool().run(n, [&](int t) {
            const int64_t lo = pages * t / n, hi = pages * (t + 1) / n;
            for (int64_t p = lo; p < hi; ++p) {
                const int64_t off = std::min(p * kPage, bytes - 1);
                base[off] = base[off];
            }
        });
    });
}

int mdrt_host_copy(void* dst, const void* src, int64_t bytes, int32_t threads) {
    return guarded([&] {
        need((dst && src) || bytes == 0, "NULL argument");
        need(bytes >= 0 && threads >= 1 && threads <= 256, "bad host_copy arguments");
        if (bytes == 0) return;
        const int n = static_cast<int>(std::min<int64_t>(threads, std::max<int64_t>(1, bytes >> 20)));
        char* d = static_cast<char*>(dst);
        const char* sp = static_cast<const char*>(src);
        host_pool().run(n, [&](int t) {
            // 4 KB-aligned slices: every page is written (and first touched) by one thread
            const int64_t lo = (bytes * t / n) & ~int64_t(4095), hi = t + 1 == n ? bytes : (bytes * (t + 1) / n) & ~int64_t(4095);
            if (hi > lo) std::memcpy(d + lo, sp + lo, static_cast<size_t>(hi - lo));
        });
    });
}

static_assert(sizeof(cudaIpcMemHandle_t) == MDRT_IPC_HANDLE_BYTES, "IPC handle size");

int mdrt_peer_alloc(int32_t device, int64_t bytes, void** dptr, uint8_t* handle) {
    return guarded([&] {
        need(dptr && handle && bytes > 0, "bad peer_alloc arguments");
        CK(cudaSetDevice(device));
        void* p = nullptr;
        CK(cudaMalloc(&p, static_cast<size_t>(bytes)));
        cudaIpcMemHandle_t h;
        const cudaError_t e = cudaIpcGetMemHandle(&h, p);
        if (e != cudaSuccess) {
            cudaFree(p);
            CK(e);
        }
        std::memcpy(handle, &h, sizeof(h));
        *dptr = p;
    });
}

int mdrt_peer_open(int32_t device, const uint8_t* handle, void** dptr) {
    return guarded([&] {
        need(dptr && handle, "bad peer_open arguments");
        CK(cudaSetDevice(device));
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof(h));
        CK(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
    });
}

int mdrt_peer_close(void* dptr) {
    return guarded([&] {
        need(dptr != nullptr, "dptr is NULL");
        CK(cudaIpcCloseMemHandle(dptr));
    });
}

int mdrt_peer_free(void* dptr) {
    return guarded([&] {
        need(dptr != nullptr, "dptr is NULL");
        CK(cudaFree(dptr));
    });
}

int mdrt_sync(mdrt_ctx* ctx) {
    return guarded([&] {
        need(ctx != nullptr, "ctx is NULL");
        ctx->use_device();
        CK(cudaDeviceSynchronize());
    });
}

}  // extern "C"
