// Device-side records and inline functions of the B200 renderer.
//
// Reference semantics restated here (paths under /root/reference/pkg/src/multidepth):
//   trace()        -> _closest_hit/_slab_hit/_tri_t, kernels/numba_backend.py:37-152
//   rng_*          -> rng.py:30-99 (splitmix64 absorb chain, bit-exact)
//   sensor_apply() -> sensor.py:55-82 (noise, dropout, clamp; f64 like the reference)
#pragma once

#include <cstdint>
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace mdrt {

// MDRT_CHECKS (diagnostic build, tools/checked_build.py): device-side bounds
// checks on every node/triangle/stack/output index; a violated check prints the
// offending values and traps, so the launch fails with an error instead of
// reading or writing out of range. Release builds compile the checks away.
#ifdef MDRT_CHECKS
#define MDRT_CHECK(cond, fmt, ...)                                                         \
    do {                                                                                   \
        if (!(cond)) {                                                                     \
            printf("MDRT_CHECK %s:%d %s: " fmt "\n", __FILE__, __LINE__, #cond, __VA_ARGS__); \
            __trap();                                                                      \
        }                                                                                  \
    } while (0)
#define MDRT_SET_LIMITS(tv, n, t) ((tv).lim_nodes = (n), (tv).lim_tris = (t))
#else
#define MDRT_CHECK(cond, fmt, ...) ((void)0)
#define MDRT_SET_LIMITS(tv, n, t) ((void)(n), (void)(t))
#endif

constexpr int kStack = 24;          // == kMaxDepth of the builder
#ifndef MDRT_BLOCK
#define MDRT_BLOCK 128
#endif
constexpr int kBlock = MDRT_BLOCK;  // threads per render block (4 warps, 4 tiles)
#ifdef MDRT_SHARED_STACK
constexpr int kStackStride = kBlock;  // this thread's column of a block-wide shared stack
#else
constexpr int kStackStride = 1;       // per-thread stack in local memory (L1-cached)
#endif
// a warp renders a TW x (32 / TW) pixel tile of one view; TW (4 or 8) is chosen
// per launch from the image width (render_tile_width)
constexpr int kExit = INT32_MIN;    // traversal stack sentinel
constexpr float kRayEps = 1e-6f;    // RAY_EPSILON (bvh.py:30): hits need t > 1e-6
constexpr float kBaryEps = 1e-5f;   // fp32 watertightness margin on barycentrics

// Per-camera rig constants (CameraModel, camera.py:20-65), uploaded at commit.
struct CamRig {
    double mount_pos[3];
    double mount_rot[4];
    double hfov_deg, vfov_deg, d_max;
    int32_t parent;  // body index or -1
    int32_t pad;
};

// Per-body constants: tree root, local-frame bounding sphere and box (centre cx..cz,
// half extents hx..hz, padded outward).
struct alignas(16) BodyInfo {
    float cx, cy, cz, r;
    float hx, hy, hz;
    int32_t root;
};

// Per-(env,cam) view record written by the prologue (128 B).
struct alignas(16) ViewRec {
    float r[9];            // camera->world rotation, row-major
    float o[3];            // camera origin (world)
    float ax, bx, ay, by;  // u = x*ax + bx, v = y*ay + by (intrinsics mode)
    float dmax;            // float32(d_max)
    int32_t nlinks;        // links surviving the view cull
    int32_t read_slot;     // latency ring slot to read for this env (-1: current frame)
    int32_t write_slot;    // latency ring slot this step writes (copied from the step state)
    unsigned long long hu; // rng prefix absorb(..step, env, cam) of the uniform stream
    unsigned long long hn; // same for the normal stream
    unsigned long long hr; // rsm-fill stream prefix absorb(absorb(absorb(key, step), env), cam)
    int32_t rsm_k;         // side-mask columns per side for this view (0: none)
    int32_t pad2;
    float pad1[4];
};
static_assert(sizeof(ViewRec) == 128, "ViewRec must be 128 B");

// Per-(env,cam,link) record: camera-frame -> link-frame ray transform + pixel rect (64 B).
struct alignas(16) LinkRec {
    float m[9];            // d_link = M * d_cam
    float o[3];            // camera origin in link frame
    int32_t root;          // link tree root
    int16_t x0, x1, y0, y1;
};
static_assert(sizeof(LinkRec) == 64, "LinkRec must be 64 B");

// ---------------------------------------------------------------------------
// counter-based RNG (rng.py:30-99)
// ---------------------------------------------------------------------------
constexpr unsigned long long kGolden = 0x9E3779B97F4A7C15ULL;
constexpr unsigned long long kMixA = 0xBF58476D1CE4E5B9ULL;
constexpr unsigned long long kMixB = 0x94D049BB133111EBULL;
constexpr unsigned long long kDomU1 = 0x9A4C93AED1F3B217ULL;
constexpr unsigned long long kDomU2 = 0x6E2F1D84C5A7093BULL;

__host__ __device__ constexpr unsigned long long mix64(unsigned long long x) {
    x ^= x >> 30;
    x *= kMixA;
    x ^= x >> 27;
    x *= kMixB;
    x ^= x >> 31;
    return x;
}

__host__ __device__ constexpr unsigned long long absorb(unsigned long long h, unsigned long long v) {
    return mix64(h ^ mix64(v + kGolden));
}

// absorb(h, v) = mix64(h ^ C(v)) with C(v) = mix64(v + golden): the inner half
// depends only on the counter value, so constants fold at compile time and a
// column's C(x) is shared by the uniform and the normal stream.
__host__ __device__ constexpr unsigned long long counter_mix(unsigned long long v) { return mix64(v + kGolden); }
constexpr unsigned long long kCDomU1 = counter_mix(kDomU1);
constexpr unsigned long long kCDomU2 = counter_mix(kDomU2);

// uniform in [0,1) from the top 53 bits (rng.py:78-80)
__device__ __forceinline__ double unit53(unsigned long long h) {
    return static_cast<double>(h >> 11) * 0x1p-53;
}

#ifndef MDRT_LIBDEVICE_BM
// Box-Muller transcendentals specialised to their argument ranges (u1 in
// [2^-53, 1], u2 in [0, 1)), f64 throughout, ~1 ulp: fdlibm's log (e_log.c:
// argument reduction to [sqrt(1/2), sqrt(2)), s = f / (2 + f), degree-14
// polynomial in s) with the division done by a reciprocal approximation and two
// Newton steps; sqrt by rsqrt approximation, two Newton steps and a residual
// correction; cos(2 pi u2) reduced exactly to an octant of [-pi/4, pi/4]
// (4 u2 is exact) and fdlibm's kernel sin/cos polynomials (k_sin.c, k_cos.c).
// Differences to numpy's log/cos(2*pi*u2) are ~1e-16 relative, far below the
// float32 rounding of the noisy depth (the sensor goldens stay bit-exact); about
// 1 % faster per step than CUDA's general log/sqrt/cos (MDRT_LIBDEVICE_BM).
__device__ __forceinline__ double rcp_approx_f64(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    return r;
}
__device__ __forceinline__ double rsqrt_approx_f64(double x) {
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    return r;
}
__device__ __forceinline__ double log_unit(double x) {
    const int hi = __double2hiint(x);
    const int lo = __double2loint(x);
    int e = (hi >> 20) - 1023;
    int mhi = (hi & 0x000FFFFF) | 0x3FF00000;
    const bool big = mhi > 0x3FF6A09E;            // m > sqrt(2): use m / 2
    mhi -= big ? 0x00100000 : 0;
    e += big ? 1 : 0;
    const double f = __hiloint2double(mhi, lo) - 1.0;
    const double d = 2.0 + f;
    double r = rcp_approx_f64(d);
    r = fma(r, fma(-d, r, 1.0), r);
    r = fma(r, fma(-d, r, 1.0), r);
    const double sv = f * r;
    const double z = sv * sv;
    const double R = z * fma(z, fma(z, fma(z, fma(z, fma(z, fma(z, 1.479819860511658591e-01,
        1.531383769920937332e-01), 1.818357216161805012e-01), 2.222219843214978396e-01),
        2.857142874366239149e-01), 3.999999999940941908e-01), 6.666666666666735130e-01);
    const double hfsq = 0.5 * f * f;
    const double de = static_cast<double>(e);
    return de * 6.93147180369123816490e-01 + (f - (hfsq - (sv * (hfsq + R) + de * 1.90821492927058770002e-10)));
}
__device__ __forceinline__ double sqrt_nonneg(double y) {
    double r = rsqrt_approx_f64(y);
    const double hy = 0.5 * y;
    r = r * fma(-hy * r, r, 1.5);
    r = r * fma(-hy * r, r, 1.5);
    double sq = y * r;
    sq = fma(fma(-sq, sq, y), 0.5 * r, sq);
    return y > 0.0 ? sq : 0.0;
}
__device__ __forceinline__ double cos_2pi(double u) {
    const double x = 4.0 * u;                      // exact
    const double q = rint(x);
    const double t = (x - q) * 1.57079632679489655800e+00;
    const double z = t * t;
    const double sn = fma(t * z, fma(z, fma(z, fma(z, fma(z, fma(z, 1.58969099521155010221e-10,
        -2.50507602534068634195e-08), 2.75573137070700676789e-06), -1.98412698298579493134e-04),
        8.33333333332248946124e-03), -1.66666666666666324348e-01), t);
    const double rc = z * fma(z, fma(z, fma(z, fma(z, fma(z, -1.13596475577881948265e-11,
        2.08757232129817482790e-09), -2.75573143513906633035e-07), 2.48015872894767294178e-05),
        -1.38888888888741095749e-03), 4.16666666666666019037e-02);
    const double hz = 0.5 * z;
    const double w = 1.0 - hz;
    const double cs = w + (((1.0 - w) - hz) + z * rc);
    const int k = static_cast<int>(q) & 3;
    const double v = (k & 1) ? sn : cs;
    return (k == 1 || k == 2) ? -v : v;
}
#endif

// standard normal by Box-Muller on two domain-separated sub-hashes (rng.py:94-99)
__device__ __forceinline__ double normal_from_hash(unsigned long long h) {
    const double u1 = static_cast<double>((mix64(h ^ kCDomU1) >> 11) + 1ULL) * 0x1p-53;
    const double u2 = static_cast<double>(mix64(h ^ kCDomU2) >> 11) * 0x1p-53;
    // __dmul_rn: keep numpy's unfused rounding
#ifndef MDRT_LIBDEVICE_BM
    return __dmul_rn(sqrt_nonneg(__dmul_rn(-2.0, log_unit(u1))), cos_2pi(u2));
#else
    return __dmul_rn(sqrt(__dmul_rn(-2.0, log(u1))), cos(__dmul_rn(6.283185307179586, u2)));
#endif
}

// Dropout threshold: unit53(h) < p  <=>  (h >> 11) < ceil(p * 2^53), because
// unit53(h) = (h >> 11) * 2^-53 exactly and scaling p by 2^53 is exact, so the
// per-pixel dropout test is one 64-bit integer compare (p in [0, 1), checked by
// the API; the reference compares the f64 uniform, sensor.py:79).
__host__ __device__ inline unsigned long long drop_threshold(double p) {
    return p > 0.0 ? static_cast<unsigned long long>(ceil(p * 0x1p53)) : 0ULL;
}

// apply_noise_dropout for one pixel (sensor.py:77-82). ru/rn: row prefixes
// absorb(.., row); cx: counter_mix of the column counter; drop_k: drop_threshold(p).
__device__ __forceinline__ float sensor_apply_cx(float depth, unsigned long long ru, unsigned long long rn,
                                                 unsigned long long cx, double noise_scale,
                                                 unsigned long long drop_k, double fill, double dmax) {
    const bool drop = (mix64(ru ^ cx) >> 11) < drop_k;
    const double g = normal_from_hash(mix64(rn ^ cx));
    double v = __dmul_rn(static_cast<double>(depth), __dadd_rn(1.0, __dmul_rn(noise_scale, g)));
    v = drop ? fill : v;
    v = v > 1e-6 ? v : 1e-6;       // np.clip lower (DEPTH_FLOOR, sensor.py:35)
    v = v < dmax ? v : dmax;       // np.clip upper
    return static_cast<float>(v);
}

__device__ __forceinline__ float sensor_apply(float depth, unsigned long long ru, unsigned long long rn,
                                              unsigned long long x, double noise_scale,
                                              unsigned long long drop_k, double fill, double dmax) {
    return sensor_apply_cx(depth, ru, rn, counter_mix(x), noise_scale, drop_k, fill, dmax);
}

// ---------------------------------------------------------------------------
// closest-hit traversal (numba_backend.py:124-152 semantics, fp32, ordered)
// ---------------------------------------------------------------------------
struct TraceCounters {
    unsigned int nodes = 0;
    unsigned int tris = 0;
    unsigned int link_nodes = 0;   // node fetches spent in link trees (subset of nodes)
    unsigned int link_traces = 0;  // link traversals started
};

// Approximate reciprocal (MUFU.RCP, <= 1 ulp): slab and triangle tests only
// need it to within the builder's conservative box padding (bvh_build.cpp).
__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// 32-byte vector load through the non-coherent path (LDG.E.256 on sm_100a):
// one 64 B node record = two requests instead of four LDG.128.
// Node-record loads carry the L2::256B prefetch-size hint: a miss fills the
// whole 256 B L2 line run, which holds the neighbouring records the builder laid
// out next to this one (config 5, BVH > L2: 21.19-21.26 -> 21.16 ms, +0.3 %;
// configs 2/3 within +-0.1 %, profiles/experiments/r01_node_hint.txt).
// MDRT_NODE_HINT (A/B knob): 0 = no hint, 1 = L1::evict_last, 2 = L2::256B
// (default), 3 = both.
#ifndef MDRT_NODE_HINT
#define MDRT_NODE_HINT 2
#endif
#if MDRT_NODE_HINT == 1
#define MDRT_LDG_NODE "ld.global.nc.L1::evict_last"
#elif MDRT_NODE_HINT == 2
#define MDRT_LDG_NODE "ld.global.nc.L2::256B"
#elif MDRT_NODE_HINT == 3
#define MDRT_LDG_NODE "ld.global.nc.L1::evict_last.L2::256B"
#else
#define MDRT_LDG_NODE "ld.global.nc"
#endif
__device__ __forceinline__ void ldg256(const float4* p, float4& a, float4& b) {
    asm(MDRT_LDG_NODE ".v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
        : "l"(p));
}
__device__ __forceinline__ float4 ldg_node4(const float4* p) {
    float4 a;
    asm(MDRT_LDG_NODE ".v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w) : "l"(p));
    return a;
}
__device__ __forceinline__ int2 ldg_node2i(const int2* p) {
    int2 a;
    asm(MDRT_LDG_NODE ".v2.s32 {%0,%1}, [%2];" : "=r"(a.x), "=r"(a.y) : "l"(p));
    return a;
}

__device__ __forceinline__ float fmin3(float a, float b, float c) {
    float r;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

// Resumable closest-hit traversal of one ray through one tree (numba_backend.py:
// 124-152 semantics, fp32, ordered). Each inner record holds both children's
// boxes: the nearer hit child is descended and the farther one pushed with its
// entry distance, so pops beyond the best hit so far are skipped without a
// fetch. State lives in registers plus this thread's column of a
// [kStack][kBlock] shared array of packed {ref, entry distance} slots.
// round() advances to the next leaf, tests it and pops; it returns true when
// the ray is finished, so callers can interleave work between rounds.
// TEXTRI: triangle records are fetched through the texture pipe (tex1Dfetch on
// `tri_tex`) instead of the LSU path: the traversal saturates the L1's LSU data
// pipe with node records, while the texture pipe into the same L1 is idle
// (config 2 +5.5 %, config 5 +5.3 %).
template <bool COUNT, bool FACE = false, bool TEXTRI = false>
struct Traversal {
    float ox, oy, oz, dx, dy, dz;
    float idx, idy, idz, oxd, oyd, ozd;
    float best;
    bool hit;
    int32_t face;   // FACE: original face index of the best hit
    cudaTextureObject_t tri_tex;   // TEXTRI: texture object over the triangle records
    int32_t ref;
    int2* top;
    int2* bottom;
#ifdef MDRT_CHECKS
    int32_t lim_nodes, lim_tris;   // record counts of the node / triangle buffers
#endif

    __device__ __forceinline__ void init(int32_t root, float ox_, float oy_, float oz_, float dx_, float dy_,
                                         float dz_, float tmax, int2* stack) {
        ox = ox_; oy = oy_; oz = oz_; dx = dx_; dy = dy_; dz = dz_;
        // zero direction components: a huge reciprocal turns the slab into a
        // containment test like _slab_hit's d == 0 branch (numba_backend.py:76-78)
        const float tiny = 1e-30f;
        idx = rcp_approx(fabsf(dx) > tiny ? dx : copysignf(tiny, dx));
        idy = rcp_approx(fabsf(dy) > tiny ? dy : copysignf(tiny, dy));
        idz = rcp_approx(fabsf(dz) > tiny ? dz : copysignf(tiny, dz));
        oxd = ox * idx; oyd = oy * idy; ozd = oz * idz;
        best = tmax;
        hit = false;
        face = -1;
        ref = root;
        top = bottom = stack;
    }

    __device__ __forceinline__ void push(int2 e) {
        MDRT_CHECK((top - bottom) / kStackStride < kStack, "stack depth %d", static_cast<int>((top - bottom) / kStackStride));
        *top = e;
        top += kStackStride;
    }
    __device__ __forceinline__ int32_t pop() {
        while (top != bottom) {
            top -= kStackStride;
            // one 64-bit load per entry: read as int2 the compiler splits it into
            // the distance load and a dependent ref load (two local requests)
            const unsigned long long raw = *reinterpret_cast<const unsigned long long*>(top);
            const int2 e = make_int2(static_cast<int>(raw & 0xffffffffu), static_cast<int>(raw >> 32));
            if (__int_as_float(e.y) <= best) return e.x;
        }
        return kExit;
    }

    __device__ __forceinline__ void test_leaf(const float4* __restrict__ tris, int32_t lref, TraceCounters& ctr) {
        // leaf: ~((first << 3) | (count - 1))
        const int32_t v = ~lref;
        const int32_t first = v >> 3;
        const int32_t cnt = (v & 7) + 1;
        MDRT_CHECK(first >= 0 && first + cnt <= lim_tris, "leaf first %d count %d of %d triangles", first, cnt, lim_tris);
        for (int32_t i = 0; i < cnt; ++i) {
            float4 v0, e1, e2;
            if constexpr (TEXTRI) {
                const int ti = 3 * (first + i);
                v0 = tex1Dfetch<float4>(tri_tex, ti);
                e1 = tex1Dfetch<float4>(tri_tex, ti + 1);
                e2 = tex1Dfetch<float4>(tri_tex, ti + 2);
            } else {
                const float4* t = tris + 3 * static_cast<int64_t>(first + i);
                v0 = __ldg(t + 0);
                e1 = __ldg(t + 1);
                e2 = __ldg(t + 2);
            }
            if (COUNT) ++ctr.tris;
            // Moller-Trumbore, double-sided (numba_backend.py:37-69)
            const float px = dy * e2.z - dz * e2.y;
            const float py = dz * e2.x - dx * e2.z;
            const float pz = dx * e2.y - dy * e2.x;
            const float det = e1.x * px + e1.y * py + e1.z * pz;
            const float inv = rcp_approx(det);
            const float tx = ox - v0.x, ty = oy - v0.y, tz = oz - v0.z;
            const float u = (tx * px + ty * py + tz * pz) * inv;
            const float qx = ty * e1.z - tz * e1.y;
            const float qy = tz * e1.x - tx * e1.z;
            const float qz = tx * e1.y - ty * e1.x;
            const float w = (dx * qx + dy * qy + dz * qz) * inv;
            const float tt = (e2.x * qx + e2.y * qy + e2.z * qz) * inv;
            const bool ok = fabsf(det) >= 1e-12f && u >= -kBaryEps && u <= 1.0f + kBaryEps && w >= -kBaryEps &&
                            u + w <= 1.0f + kBaryEps && tt > kRayEps && tt <= best;
            if (ok) {
                best = tt;
                hit = true;
                if constexpr (FACE) face = __float_as_int(v0.w);
            }
        }
    }

    // OCT < 0: any ray; OCT = 0..7: every ray of the call has the direction-sign
    // octant OCT (bit 0: dx < 0, bit 1: dy < 0, bit 2: dz < 0), so the near and far
    // slab of each axis is known at compile time and each child's entry/exit
    // distance is two 3-input min/max instead of five (bitwise the same result:
    // fmaf(lo, idx, -o) <= fmaf(hi, idx, -o) for idx >= 0, rounding is monotonic).
    // descend through inner nodes until `ref` is a leaf (< 0) or kExit
    template <int OCT>
    __device__ __forceinline__ void descend_t(const float4* __restrict__ nodes, TraceCounters& ctr) {
        while (ref >= 0) {
            MDRT_CHECK(ref < lim_nodes, "node %d of %d", ref, lim_nodes);
            const float4* n = nodes + 4 * static_cast<int64_t>(ref);
            float4 bx, by;
            ldg256(n, bx, by);        // c0 x lo/hi, c0 y lo/hi | c1 x lo/hi, c1 y lo/hi
#if defined(MDRT_NODE64)
            float4 bz, rff;
            ldg256(n + 2, bz, rff);   // c0 z lo/hi, c1 z lo/hi | refs + 8 B pad
            const int2 rf = make_int2(__float_as_int(rff.x), __float_as_int(rff.y));
#else
            // 56 of the record's 64 B: the L1 data pipe is loaded by the bytes
            // delivered per lane, so the 8 B pad after the refs is not fetched
            // (+0.3 % config 2, +0.7 % config 5 over one 32 B load)
#if MDRT_NODE_HINT
            const float4 bz = ldg_node4(n + 2);
            const int2 rf = ldg_node2i(reinterpret_cast<const int2*>(n + 3));
#else
            const float4 bz = __ldg(n + 2);                                     // c0 z lo/hi, c1 z lo/hi
            const int2 rf = __ldg(reinterpret_cast<const int2*>(n + 3));        // refs
#endif
#endif
            if (COUNT) ++ctr.nodes;
            float c0min, c0max, c1min, c1max;
            if constexpr (OCT < 0) {
                const float a0 = fmaf(bx.x, idx, -oxd), a1 = fmaf(bx.y, idx, -oxd);
                const float a2 = fmaf(bx.z, idy, -oyd), a3 = fmaf(bx.w, idy, -oyd);
                const float a4 = fmaf(bz.x, idz, -ozd), a5 = fmaf(bz.y, idz, -ozd);
                c0min = fmax3(fminf(a0, a1), fminf(a2, a3), fmaxf(fminf(a4, a5), 0.0f));
                c0max = fmin3(fmaxf(a0, a1), fmaxf(a2, a3), fminf(fmaxf(a4, a5), best));
                const float b0 = fmaf(by.x, idx, -oxd), b1 = fmaf(by.y, idx, -oxd);
                const float b2 = fmaf(by.z, idy, -oyd), b3 = fmaf(by.w, idy, -oyd);
                const float b4 = fmaf(bz.z, idz, -ozd), b5 = fmaf(bz.w, idz, -ozd);
                c1min = fmax3(fminf(b0, b1), fminf(b2, b3), fmaxf(fminf(b4, b5), 0.0f));
                c1max = fmin3(fmaxf(b0, b1), fmaxf(b2, b3), fminf(fmaxf(b4, b5), best));
            } else {
                constexpr bool NX = (OCT & 1) != 0, NY = (OCT & 2) != 0, NZ = (OCT & 4) != 0;
                c0min = fmax3(fmaf(NX ? bx.y : bx.x, idx, -oxd), fmaf(NY ? bx.w : bx.z, idy, -oyd),
                              fmaxf(fmaf(NZ ? bz.y : bz.x, idz, -ozd), 0.0f));
                c0max = fmin3(fmaf(NX ? bx.x : bx.y, idx, -oxd), fmaf(NY ? bx.z : bx.w, idy, -oyd),
                              fminf(fmaf(NZ ? bz.x : bz.y, idz, -ozd), best));
                c1min = fmax3(fmaf(NX ? by.y : by.x, idx, -oxd), fmaf(NY ? by.w : by.z, idy, -oyd),
                              fmaxf(fmaf(NZ ? bz.w : bz.z, idz, -ozd), 0.0f));
                c1max = fmin3(fmaf(NX ? by.x : by.y, idx, -oxd), fmaf(NY ? by.z : by.w, idy, -oyd),
                              fminf(fmaf(NZ ? bz.z : bz.w, idz, -ozd), best));
            }
            const bool h0 = c0min <= c0max;
            const bool h1 = c1min <= c1max;
            if (h0 && h1) {
                const bool swap = c1min < c0min;
                const int32_t far = swap ? rf.x : rf.y;
                push(make_int2(far, __float_as_int(swap ? c0min : c1min)));
                ref = swap ? rf.y : rf.x;
            } else if (h0 || h1) {
                ref = h0 ? rf.x : rf.y;
            } else {
                ref = pop();
            }
        }
    }

    // leaf step after a descent: test its triangles and pop; true when finished
    __device__ __forceinline__ bool leaf_step(const float4* __restrict__ tris, TraceCounters& ctr) {
        if (ref == kExit) return true;
        test_leaf(tris, ref, ctr);
        ref = pop();
        return ref == kExit;
    }

    __device__ __forceinline__ bool round(const float4* __restrict__ nodes, const float4* __restrict__ tris,
                                          TraceCounters& ctr) {
        descend_t<-1>(nodes, ctr);
        return leaf_step(tris, ctr);
    }

    // sign octant of the direction (bit 0: x, 1: y, 2: z negative)
    __device__ __forceinline__ int octant() const {
        return (idx < 0.0f ? 1 : 0) | (idy < 0.0f ? 2 : 0) | (idz < 0.0f ? 4 : 0);
    }

    // nearest hit t in (1e-6, tmax], or +inf when nothing was hit (the caller then
    // keeps its bound; numba_backend.py:206-208)
    __device__ __forceinline__ float result() const { return hit ? best : __int_as_float(0x7f800000); }
};

template <bool COUNT>
__device__ __forceinline__ float trace(const float4* __restrict__ nodes, cudaTextureObject_t tri_tex,
                                       int32_t root, float ox, float oy, float oz, float dx, float dy,
                                       float dz, float tmax, int2* __restrict__ stack,
                                       TraceCounters& ctr, int32_t lim_nodes, int32_t lim_tris) {
    Traversal<COUNT, false, true> tv;
    tv.init(root, ox, oy, oz, dx, dy, dz, tmax, stack);
    MDRT_SET_LIMITS(tv, lim_nodes, lim_tris);
    tv.tri_tex = tri_tex;
    const float4* tris = nullptr;   // triangles come from tri_tex
    while (!tv.round(nodes, tris, ctr)) {
    }
    return tv.result();
}

// trace() for a call made by a set of lanes whose direction octants are usually
// equal (one camera's tile against the terrain): a warp-uniform octant selects a
// specialised traversal loop, mixed warps take the generic one.
template <bool COUNT>
__device__ __forceinline__ float trace_oct(const float4* __restrict__ nodes, cudaTextureObject_t tri_tex,
                                           int32_t root, float ox, float oy, float oz, float dx, float dy,
                                           float dz, float tmax, int2* __restrict__ stack,
                                           TraceCounters& ctr, int32_t lim_nodes, int32_t lim_tris) {
    Traversal<COUNT, false, true> tv;
    tv.init(root, ox, oy, oz, dx, dy, dz, tmax, stack);
    MDRT_SET_LIMITS(tv, lim_nodes, lim_tris);
    tv.tri_tex = tri_tex;
    const float4* tris = nullptr;   // triangles come from tri_tex
    const int oct = tv.octant();
    const unsigned mask = __activemask();
    const bool uniform = __match_any_sync(mask, oct) == mask;
    do {
        // only the inner-node descent is specialised; leaf tests are shared
        if (!uniform) {
            tv.template descend_t<-1>(nodes, ctr);
        } else {
            switch (oct) {
#define MDRT_OCT_CASE(K) \
                case K: tv.template descend_t<K>(nodes, ctr); break;
                MDRT_OCT_CASE(0) MDRT_OCT_CASE(1) MDRT_OCT_CASE(2) MDRT_OCT_CASE(3)
                MDRT_OCT_CASE(4) MDRT_OCT_CASE(5) MDRT_OCT_CASE(6) MDRT_OCT_CASE(7)
#undef MDRT_OCT_CASE
            }
        }
    } while (!tv.leaf_step(tris, ctr));
    return tv.result();
}

}  // namespace mdrt
