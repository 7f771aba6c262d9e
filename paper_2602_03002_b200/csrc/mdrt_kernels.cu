// CUDA kernels of the B200 multi-depth renderer (sm_100a).
//
//   prologue_kernel  (K4)  per-(env,cam) camera pose + intrinsics + link cull list.
//                          Replaces Scene.camera_world_poses (scene.py:279-295),
//                          ray_grids (scene.py:304-329) and the per-ray body
//                          transform of numba_backend.py:193-202.
//   render_kernel (K1+K2+K3) one warp per 8x4 pixel tile: link traversal in link
//                          frames, terrain traversal, fused sensor epilogue and
//                          latency ring. Replaces _render_kernel
//                          (numba_backend.py:155-219), apply_noise_dropout
//                          (sensor.py:55-82) and FrameBuffer (sensor.py:103-150).
//   noise_kernel, gather_kernel, select_kernel, downsample_kernel: standalone
//                          sensor-stage operators (sensor.py:55-150).
#include "mdrt_kernels.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

namespace mdrt {

// ---------------------------------------------------------------------------
// f64 pose helpers (transforms.py:32-58, 151-156). __d*_rn keeps numpy rounding.
// ---------------------------------------------------------------------------
struct Q { double w, x, y, z; };
struct V3 { double x, y, z; };

__device__ __forceinline__ Q qnorm(Q q) {
    const double n = sqrt(__dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(q.w, q.w), __dmul_rn(q.x, q.x)),
                                              __dmul_rn(q.y, q.y)), __dmul_rn(q.z, q.z)));
    // one division and four products instead of four divisions: within 1 ulp (f64)
    // of numpy's q / n, far below the f32 rounding of the poses downstream
    const double r = 1.0 / n;
    return {q.w * r, q.x * r, q.y * r, q.z * r};
}

__device__ __forceinline__ Q qmul(Q a, Q b) {
    Q r;
    r.w = a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z;
    r.x = a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y;
    r.y = a.w * b.y - a.x * b.z + a.y * b.w + a.z * b.x;
    r.z = a.w * b.z + a.x * b.y - a.y * b.x + a.z * b.w;
    return qnorm(r);
}

__device__ __forceinline__ V3 qrot(Q q, V3 v) {
    // v + w t + q_v x t,  t = 2 q_v x v
    const double tx = 2.0 * (q.y * v.z - q.z * v.y);
    const double ty = 2.0 * (q.z * v.x - q.x * v.z);
    const double tz = 2.0 * (q.x * v.y - q.y * v.x);
    return {v.x + q.w * tx + (q.y * tz - q.z * ty), v.y + q.w * ty + (q.z * tx - q.x * tz),
            v.z + q.w * tz + (q.x * ty - q.y * tx)};
}

__device__ __forceinline__ void qmat(Q q, double m[9]) {
    const double w = q.w, x = q.x, y = q.y, z = q.z;
    m[0] = 1 - 2 * (y * y + z * z); m[1] = 2 * (x * y - w * z);     m[2] = 2 * (x * z + w * y);
    m[3] = 2 * (x * y + w * z);     m[4] = 1 - 2 * (x * x + z * z); m[5] = 2 * (y * z - w * x);
    m[6] = 2 * (x * z - w * y);     m[7] = 2 * (y * z + w * x);     m[8] = 1 - 2 * (x * x + y * y);
}

// Pose of body b in env e: the scene's (N,B,3)/(N,B,4) buffers, or a record of
// a simulator's link-state tensor (zero-copy ingestion), quaternion as wxyz.
__device__ __forceinline__ void load_pose(const PrologueParams& p, int64_t e, int b, float t[3], float q[4]) {
    if (p.link_states) {
        MDRT_CHECK(p.link_map[b] >= 0 && p.link_map[b] < p.env_stride, "body %d maps to link %d of %lld", b,
                   p.link_map[b], static_cast<long long>(p.env_stride));
        const float* r = p.link_states + (e * p.env_stride + p.link_map[b]) * p.record_stride;
        t[0] = r[p.pos_offset]; t[1] = r[p.pos_offset + 1]; t[2] = r[p.pos_offset + 2];
        const float* qq = r + p.rot_offset;
        if (p.rot_xyzw) {
            q[0] = qq[3]; q[1] = qq[0]; q[2] = qq[1]; q[3] = qq[2];
        } else {
            q[0] = qq[0]; q[1] = qq[1]; q[2] = qq[2]; q[3] = qq[3];
        }
    } else {
        const int64_t k = e * p.B + b;
        const float* bp = p.body_pos + k * 3;
        const float* bq = p.body_rot + k * 4;
        t[0] = bp[0]; t[1] = bp[1]; t[2] = bp[2];
        q[0] = bq[0]; q[1] = bq[1]; q[2] = bq[2]; q[3] = bq[3];
    }
}

// ---------------------------------------------------------------------------
// Per-tile terrain entry nodes. Every ray of a pixel tile lies inside the tile's
// view pyramid: apex at the camera, side planes through the tile's corner
// pixel-centre rays, far plane at camera depth d_max (a ray's range is at most
// d_max, so its camera-frame depth is too). Descending the terrain BVH from the
// root while only one child box meets the pyramid (1 cm margin) reaches a node
// every ray of the tile would reach first anyway: a ray's own slab test can only
// enter a box its segment meets, and the skipped siblings are >= 1 cm from every
// ray, far beyond the fp32 error of the slab and triangle tests. Starting there
// yields the identical closest hit while the coherent top-level node fetches
// (all 32 lanes reading the same records) are done once per tile by one lane of
// the prologue instead of once per ray.
// ---------------------------------------------------------------------------
struct TilePyramid {
    float lo[3], hi[3];   // AABB of the apex and the far corners
    float n[6][3], d[6];  // planes n.p + d >= 0 contain the pyramid (unit n)
};

__device__ __forceinline__ void pyramid_setup(TilePyramid& f, const float R[9], const float o[3], float u0, float u1,
                                              float v0, float v1, float far) {
    const float cu[4] = {u0, u1, u1, u0}, cv[4] = {v0, v0, v1, v1};
    float D[4][3];
    for (int k = 0; k < 4; ++k) {
        D[k][0] = R[0] * cu[k] + R[1] * cv[k] + R[2];
        D[k][1] = R[3] * cu[k] + R[4] * cv[k] + R[5];
        D[k][2] = R[6] * cu[k] + R[7] * cv[k] + R[8];
    }
    for (int a = 0; a < 3; ++a) {
        f.lo[a] = o[a];
        f.hi[a] = o[a];
        for (int k = 0; k < 4; ++k) {
            const float q = o[a] + far * D[k][a];
            f.lo[a] = fminf(f.lo[a], q);
            f.hi[a] = fmaxf(f.hi[a], q);
        }
    }
    for (int k = 0; k < 4; ++k) {
        const float* A = D[k];
        const float* B = D[(k + 1) & 3];
        const float* Cn = D[(k + 2) & 3];
        float nx = A[1] * B[2] - A[2] * B[1], ny = A[2] * B[0] - A[0] * B[2], nz = A[0] * B[1] - A[1] * B[0];
        const float inv = rsqrtf(fmaxf(nx * nx + ny * ny + nz * nz, 1e-30f));
        nx *= inv; ny *= inv; nz *= inv;
        if (nx * Cn[0] + ny * Cn[1] + nz * Cn[2] < 0.f) { nx = -nx; ny = -ny; nz = -nz; }
        f.n[k][0] = nx; f.n[k][1] = ny; f.n[k][2] = nz;
        f.d[k] = -(nx * o[0] + ny * o[1] + nz * o[2]);
    }
    const float fx = R[2], fy = R[5], fz = R[8];   // camera +z (forward) in world
    const float fo = fx * o[0] + fy * o[1] + fz * o[2];
    f.n[4][0] = fx; f.n[4][1] = fy; f.n[4][2] = fz; f.d[4] = -fo;            // in front of the camera
    f.n[5][0] = -fx; f.n[5][1] = -fy; f.n[5][2] = -fz; f.d[5] = fo + far;    // within depth d_max
}

// true when the box certainly misses the pyramid (separated by its AABB or a plane)
__device__ __forceinline__ bool pyramid_misses(const TilePyramid& f, float lx, float hx, float ly, float hy, float lz,
                                               float hz) {
    constexpr float eps = 0.01f;
    if (!(lx <= f.hi[0] + eps && hx >= f.lo[0] - eps && ly <= f.hi[1] + eps && hy >= f.lo[1] - eps &&
          lz <= f.hi[2] + eps && hz >= f.lo[2] - eps))
        return true;   // also empty boxes (lo = +inf, hi = -inf)
    const float cx = 0.5f * (lx + hx), cy = 0.5f * (ly + hy), cz = 0.5f * (lz + hz);
    const float ex = 0.5f * (hx - lx), ey = 0.5f * (hy - ly), ez = 0.5f * (hz - lz);
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        const float* n = f.n[k];
        const float reach = n[0] * cx + n[1] * cy + n[2] * cz + fabsf(n[0]) * ex + fabsf(n[1]) * ey +
                            fabsf(n[2]) * ez + f.d[k];
        if (reach < -eps) return true;
    }
    return false;
}

// Descend from the terrain root while exactly one child meets the pyramid. The
// entry is the record holding the last child descended into: a ray started there
// still tests that child's box itself (a node record holds its children's boxes,
// not its own), so rays of the tile that miss it stop exactly where a traversal
// from the root would, and the sibling box they skip is outside the pyramid.
// kExit when no terrain box meets the pyramid.
__device__ int32_t pyramid_entry(const float4* __restrict__ nodes, int32_t root, const TilePyramid& f,
                                 int32_t n_nodes) {
    int32_t rec = root;
    for (int lvl = 0; lvl <= kStack + 1; ++lvl) {
        MDRT_CHECK(rec >= 0 && rec < n_nodes, "entry descent: node %d of %d", rec, n_nodes);
        const float4* n = nodes + 4 * static_cast<int64_t>(rec);
        const float4 bx = __ldg(n), by = __ldg(n + 1), bz = __ldg(n + 2);
        const int2 rf = __ldg(reinterpret_cast<const int2*>(n + 3));
        const bool m0 = pyramid_misses(f, bx.x, bx.y, bx.z, bx.w, bz.x, bz.y);
        const bool m1 = pyramid_misses(f, by.x, by.y, by.z, by.w, bz.z, bz.w);
        if (m0 && m1) return kExit;
        if (!m0 && !m1) break;
        const int32_t child = m0 ? rf.y : rf.x;
        if (child < 0) break;   // a leaf: its box is in this record
        rec = child;
    }
    return rec;
}

// One thread per (view, tile), after the prologue wrote the view records (the
// render kernel's own f32 camera rotation, origin and intrinsics).
static __global__ void __launch_bounds__(128) entry_kernel(EntryParams p) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= p.views_count * p.tiles_per_view) return;
    const int64_t view = i / p.tiles_per_view;
    const int tl = static_cast<int>(i - view * p.tiles_per_view);
    const ViewRec& V = p.views[view];
    float R[9], o[3];
    for (int k = 0; k < 9; ++k) R[k] = V.r[k];
    for (int k = 0; k < 3; ++k) o[k] = V.o[k];
    const int ty = tl / p.tiles_x, tx = tl - ty * p.tiles_x;
    const int x0 = tx * p.tile_w, x1 = min(x0 + p.tile_w, p.W) - 1;
    const int y0 = ty * p.tile_h, y1 = min(y0 + p.tile_h, p.H) - 1;
    constexpr float m = 1e-4f;   // direction margin (tangent units) over the f32 rounding of u, v
    TilePyramid f;
    pyramid_setup(f, R, o, fmaf(static_cast<float>(x0), V.ax, V.bx) - m, fmaf(static_cast<float>(x1), V.ax, V.bx) + m,
                  fmaf(static_cast<float>(y0), V.ay, V.by) - m, fmaf(static_cast<float>(y1), V.ay, V.by) + m, V.dmax);
    p.out[i] = pyramid_entry(p.nodes, p.root, f, p.n_nodes);
}

// ---------------------------------------------------------------------------
// K4 prologue: one warp per (env, cam); lanes walk the links.
// ---------------------------------------------------------------------------
#ifndef MDRT_PRO_MINB
#define MDRT_PRO_MINB 8   // 64 registers: 4x the resident warps of the unbounded 133-register build;
                          // the f64 pose chain is latency-bound (53 -> 32 us at config 2)
#endif
static __global__ void __launch_bounds__(128, MDRT_PRO_MINB) prologue_kernel(PrologueParams p) {
    const int lane = threadIdx.x & 31;
    const int64_t view = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (view >= static_cast<int64_t>(p.N) * p.C) return;
    const int e = static_cast<int>(view / p.C);
    const int c = static_cast<int>(view - static_cast<int64_t>(e) * p.C);
    const CamRig rig = p.rigs[c];

    // ---- camera world pose (scene.py:279-295) ----
    V3 t;
    Q q;
    if (p.cam_pos) {
        const float* cp = p.cam_pos + view * 3;
        const float* cq = p.cam_rot + view * 4;
        t = {cp[0], cp[1], cp[2]};
        q = {cq[0], cq[1], cq[2], cq[3]};
    } else {
        t = {rig.mount_pos[0], rig.mount_pos[1], rig.mount_pos[2]};
        q = {rig.mount_rot[0], rig.mount_rot[1], rig.mount_rot[2], rig.mount_rot[3]};
        if (rig.parent >= 0) {
            float bp[3], bq[4];
            load_pose(p, e, rig.parent, bp, bq);
            Q pq = qnorm(qnorm({bq[0], bq[1], bq[2], bq[3]}));
            V3 rt = qrot(pq, t);
            t = {bp[0] + rt.x, bp[1] + rt.y, bp[2] + rt.z};
            q = qnorm(qmul(pq, q));
        }
        if (p.off_pos) {
            const float* op = p.off_pos + view * 3;
            const float* oq = p.off_rot + view * 4;
            Q offq = qnorm(qnorm({oq[0], oq[1], oq[2], oq[3]}));
            V3 rt = qrot(q, {op[0], op[1], op[2]});
            t = {t.x + rt.x, t.y + rt.y, t.z + rt.z};
            q = qnorm(qmul(q, offq));
        }
    }
    double R[9];
    qmat(q, R);

    // ---- intrinsics (camera.py:51-65, with_fov_delta camera.py:92-95) ----
    const double delta = p.fov_delta ? static_cast<double>(p.fov_delta[view]) : 0.0;
    const double kDeg = 3.141592653589793 / 180.0;
    const double fx = (p.W / 2.0) / tan(((rig.hfov_deg + delta) * kDeg) / 2.0);
    const double fy = (p.H / 2.0) / tan(((rig.vfov_deg + delta) * kDeg) / 2.0);
    const double cx = p.W / 2.0, cy = p.H / 2.0;
    const bool grid = p.grid_mode;

    // ---- link cull list (f32: conservative to well under a pixel; M and o are
    // rounded to f32 for the traversal anyway) ----
    float Rf[9];
    for (int i = 0; i < 9; ++i) Rf[i] = static_cast<float>(R[i]);
    const float fxf = static_cast<float>(fx), fyf = static_cast<float>(fy);
    const float cxf = static_cast<float>(cx), cyf = static_cast<float>(cy);
    int count = 0;
    for (int base = 0; base < p.B; base += 32) {
        const int b = base + lane;
        bool keep = false;
        LinkRec rec;
        if (b < p.B) {
            const BodyInfo bi = p.bodies[b];
            float bp[3], bq[4];
            load_pose(p, e, b, bp, bq);
            float qw = bq[0], qx = bq[1], qy = bq[2], qz = bq[3];
            const float qn = rsqrtf(qw * qw + qx * qx + qy * qy + qz * qz);
            qw *= qn; qx *= qn; qy *= qn; qz *= qn;
            const float L[9] = {1.f - 2.f * (qy * qy + qz * qz), 2.f * (qx * qy - qw * qz), 2.f * (qx * qz + qw * qy),
                                2.f * (qx * qy + qw * qz), 1.f - 2.f * (qx * qx + qz * qz), 2.f * (qy * qz - qw * qx),
                                2.f * (qx * qz - qw * qy), 2.f * (qy * qz + qw * qx), 1.f - 2.f * (qx * qx + qy * qy)};
            // camera origin relative to the link origin (f64 difference, then f32)
            const float ox = static_cast<float>(t.x - bp[0]);
            const float oy = static_cast<float>(t.y - bp[1]);
            const float oz = static_cast<float>(t.z - bp[2]);
            // link-box centre relative to the camera, camera frame
            const float wx = L[0] * bi.cx + L[1] * bi.cy + L[2] * bi.cz - ox;
            const float wy = L[3] * bi.cx + L[4] * bi.cy + L[5] * bi.cz - oy;
            const float wz = L[6] * bi.cx + L[7] * bi.cy + L[8] * bi.cz - oz;
            const float X = Rf[0] * wx + Rf[3] * wy + Rf[6] * wz;
            const float Y = Rf[1] * wx + Rf[4] * wy + Rf[7] * wz;
            const float Z = Rf[2] * wx + Rf[5] * wy + Rf[8] * wz;
            const float dist = sqrtf(X * X + Y * Y + Z * Z);
            keep = (dist - bi.r) <= static_cast<float>(rig.d_max) * (1.0f + 1e-5f) + 1e-5f;
            int x0 = 0, x1 = p.W - 1, y0 = 0, y1 = p.H - 1;
            if (keep && !grid && !p.no_cull) {
                // Project the link box (clipped at the hit plane z = 1e-6; camera-frame
                // rays are (u, v, 1) so z == t) to a conservative pixel rectangle.
                float A[3][3];  // camera-frame half-axis vectors of the box
                const float hk[3] = {bi.hx, bi.hy, bi.hz};
                for (int kx = 0; kx < 3; ++kx) {
                    const float lx = L[0 * 3 + kx] * hk[kx], ly = L[1 * 3 + kx] * hk[kx], lz = L[2 * 3 + kx] * hk[kx];
                    A[kx][0] = Rf[0] * lx + Rf[3] * ly + Rf[6] * lz;
                    A[kx][1] = Rf[1] * lx + Rf[4] * ly + Rf[7] * lz;
                    A[kx][2] = Rf[2] * lx + Rf[5] * ly + Rf[8] * lz;
                }
                float cx3[8][3];
                for (int q8 = 0; q8 < 8; ++q8) {
                    const float s0 = (q8 & 1) ? 1.f : -1.f, s1 = (q8 & 2) ? 1.f : -1.f, s2 = (q8 & 4) ? 1.f : -1.f;
                    cx3[q8][0] = X + s0 * A[0][0] + s1 * A[1][0] + s2 * A[2][0];
                    cx3[q8][1] = Y + s0 * A[0][1] + s1 * A[1][1] + s2 * A[2][1];
                    cx3[q8][2] = Z + s0 * A[0][2] + s1 * A[1][2] + s2 * A[2][2];
                }
                const float zc = 1e-6f;
                float sxlo = 3e38f, sxhi = -3e38f, sylo = 3e38f, syhi = -3e38f;
                int front = 0;
                for (int q8 = 0; q8 < 8; ++q8) {
                    if (cx3[q8][2] > zc) {
                        ++front;
                        const float iz = 1.0f / cx3[q8][2];
                        const float sx = cx3[q8][0] * iz, sy = cx3[q8][1] * iz;
                        sxlo = fminf(sxlo, sx); sxhi = fmaxf(sxhi, sx);
                        sylo = fminf(sylo, sy); syhi = fmaxf(syhi, sy);
                    }
                }
                keep = front > 0;
                if (keep && front < 8) {
                    // edges crossing the clip plane contribute their crossing point
                    for (int q8 = 0; q8 < 8; ++q8)
                        for (int bit = 1; bit < 8; bit <<= 1) {
                            const int q2 = q8 | bit;
                            if (q2 == q8) continue;
                            const float z0 = cx3[q8][2], z1 = cx3[q2][2];
                            if ((z0 > zc) == (z1 > zc)) continue;
                            const float f = (zc - z0) / (z1 - z0);
                            const float sx = (cx3[q8][0] + f * (cx3[q2][0] - cx3[q8][0])) / zc;
                            const float sy = (cx3[q8][1] + f * (cx3[q2][1] - cx3[q8][1])) / zc;
                            sxlo = fminf(sxlo, sx); sxhi = fmaxf(sxhi, sx);
                            sylo = fminf(sylo, sy); syhi = fmaxf(syhi, sy);
                        }
                }
                if (keep) {
                    const float xl = sxlo * fxf + cxf - 0.5f, xh = sxhi * fxf + cxf - 0.5f;
                    const float yl = sylo * fyf + cyf - 0.5f, yh = syhi * fyf + cyf - 0.5f;
                    x0 = xl > x0 ? static_cast<int>(fminf(floorf(xl) - 1.0f, 1e9f)) : x0;
                    x1 = xh < x1 ? static_cast<int>(fmaxf(ceilf(xh) + 1.0f, -1e9f)) : x1;
                    y0 = yl > y0 ? static_cast<int>(fminf(floorf(yl) - 1.0f, 1e9f)) : y0;
                    y1 = yh < y1 ? static_cast<int>(fmaxf(ceilf(yh) + 1.0f, -1e9f)) : y1;
                    x0 = max(x0, 0); y0 = max(y0, 0);
                    x1 = min(x1, p.W - 1); y1 = min(y1, p.H - 1);
                    keep = x0 <= x1 && y0 <= y1;
                }
            }
            if (keep) {
                // M = L^T R (camera frame -> link frame), o = L^T (t - p)
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 3; ++j)
                        rec.m[i * 3 + j] = L[0 * 3 + i] * Rf[0 * 3 + j] + L[1 * 3 + i] * Rf[1 * 3 + j] +
                                           L[2 * 3 + i] * Rf[2 * 3 + j];
                rec.o[0] = L[0] * ox + L[3] * oy + L[6] * oz;
                rec.o[1] = L[1] * ox + L[4] * oy + L[7] * oz;
                rec.o[2] = L[2] * ox + L[5] * oy + L[8] * oz;
                rec.root = bi.root;
                rec.x0 = static_cast<int16_t>(x0);
                rec.x1 = static_cast<int16_t>(x1);
                rec.y0 = static_cast<int16_t>(y0);
                rec.y1 = static_cast<int16_t>(y1);
            }
        }
        const unsigned mask = __ballot_sync(0xffffffffu, keep);
        if (keep) {
            const int slot = count + __popc(mask & ((1u << lane) - 1u));
            p.links[view * p.B + slot] = rec;
            p.rects[view * p.B + slot] = make_int2((rec.x0 & 0xffff) | (static_cast<int>(rec.x1) << 16),
                                                   (rec.y0 & 0xffff) | (static_cast<int>(rec.y1) << 16));
        }
        count += __popc(mask);
    }

    if (view == 0 && p.reset_counter)
        for (int i = lane; i < p.reset_count; i += 32) p.reset_counter[i] = 0u;

    // ---- view record ----
    if (lane == 0) {
        ViewRec v;
        for (int i = 0; i < 9; ++i) v.r[i] = static_cast<float>(R[i]);
        v.o[0] = static_cast<float>(t.x);
        v.o[1] = static_cast<float>(t.y);
        v.o[2] = static_cast<float>(t.z);
        v.ax = static_cast<float>(1.0 / fx);
        v.bx = static_cast<float>((0.5 - cx) / fx);
        v.ay = static_cast<float>(1.0 / fy);
        v.by = static_cast<float>((0.5 - cy) / fy);
        v.dmax = static_cast<float>(rig.d_max);
        v.nlinks = count;
        v.read_slot = -1;
        v.write_slot = 0;
        const unsigned long long genv = static_cast<unsigned long long>(p.env_offset + e);
        const StepState* st = p.state;
        v.hu = absorb(absorb(st ? st->hu_step : p.hu_step, genv), static_cast<unsigned long long>(c));
        v.hn = absorb(absorb(st ? st->hn_step : p.hn_step, genv), static_cast<unsigned long long>(c));
        v.rsm_k = p.rsm_modes ? p.rsm_k[min(max(p.rsm_modes[view], 0), 2)] : 0;
        v.hr = absorb(absorb(st ? st->hr_step : p.hr_step, genv), static_cast<unsigned long long>(c));
        v.pad2 = 0;
        if (p.latency) {
            // bisect_right(times, now - delay) - 1, clamped at 0 (sensor.py:138-139)
            const double* times = st ? st->times : p.ring_times;
            const int32_t* order = st ? st->order : p.ring_order;
            const int count = st ? st->ring_count : p.ring_count;
            const int wslot = st ? st->write_slot : p.write_slot;
            const double target = (st ? st->now : p.now) - p.delays[e];
            int lo = 0, hi = count;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (target < times[mid]) hi = mid;
                else lo = mid + 1;
            }
            const int kk = lo - 1 < 0 ? 0 : lo - 1;
            MDRT_CHECK(count >= 0 && count <= 32 && kk < 32, "ring count %d index %d", count, kk);
            const int slot = order[kk];
            v.read_slot = slot == wslot ? -1 : slot;
            v.write_slot = wslot;
            if (c == 0 && p.read_slot_out) p.read_slot_out[e] = slot;
        }
        for (int i = 0; i < 4; ++i) v.pad1[i] = 0.f;
        p.views[view] = v;
    }
}

// ---------------------------------------------------------------------------
// K1+K2+K3: render + fused sensor epilogue. One warp = one 8x4 tile of a view.
// ---------------------------------------------------------------------------
// n / d for 32-bit n with a host-precomputed m = floor((2^32 - 1) / d): the
// multiply-high estimate is at most one short, fixed by one compare.
__device__ __forceinline__ uint32_t fast_div(uint32_t n, uint32_t d, uint32_t m) {
    uint32_t q = __umulhi(n, m);
    if (n - q * d >= d) ++q;
    return q;
}

#ifdef MDRT_PLAIN_STORES
__device__ __forceinline__ void st_stream(float* p, float v) { *p = v; }
#else
__device__ __forceinline__ void st_stream(float* p, float v) { __stcs(p, v); }
#endif

template <bool COUNT, int TW>
__device__ __forceinline__ void render_tile(const RenderParams& p, uint32_t gw, int lane, int2* stack) {
    constexpr int kTileW = TW;          // this launch's tile shape: TW x (32 / TW) pixels
    constexpr int kTileH = 32 / TW;
    // gw -> (q1, q2, tx) by two mixed-radix divisions; view-major order has
    // q1 = view, q2 = tile row, tile-row-major order (row_order) the reverse:
    // tile row 0 of every view comes first, so the expensive rows (towards
    // the horizon) start early and the launch ends on cheap near-ground rows
    const uint32_t q1 = fast_div(gw, p.order_d1, p.order_m1);
    const uint32_t r1 = gw - q1 * p.order_d1;
    const uint32_t q2 = fast_div(r1, static_cast<uint32_t>(p.tiles_x), p.m_tiles_x);
    const uint32_t tx = r1 - q2 * static_cast<uint32_t>(p.tiles_x);
    const uint32_t view = p.row_order ? q2 : q1;
    const uint32_t ty = p.row_order ? q1 : q2;
    const int px = static_cast<int>(tx) * kTileW + (lane & (kTileW - 1));
    const int py = static_cast<int>(ty) * kTileH + lane / kTileW;
    const bool active = px < p.W && py < p.H;
    const uint32_t e = fast_div(view, static_cast<uint32_t>(p.C), p.m_C);
    const uint32_t c = view - e * static_cast<uint32_t>(p.C);
    MDRT_CHECK(view < static_cast<uint32_t>(p.N * p.C) && e < static_cast<uint32_t>(p.N) && tx < static_cast<uint32_t>(p.tiles_x),
               "tile %u: view %u env %u tx %u", gw, view, e, tx);

    const ViewRec& V = p.views[view];
    const float4 in = *reinterpret_cast<const float4*>(&V.ax);     // ax bx ay by
    const float dmax = V.dmax;
    const int nlinks = V.nlinks;
    MDRT_CHECK(nlinks >= 0 && nlinks <= p.B, "view %u nlinks %d of %d", view, nlinks, p.B);

    // camera-frame direction and scale (camera.py:81-90)
    float dcx, dcy, dcz, m;
    if (p.ray_dirs) {
        const int64_t er = p.ray_envs > 1 ? e : 0;
        const int64_t pix = ((er * p.C + c) * p.H + (active ? py : 0)) * p.W + (active ? px : 0);
        dcx = p.ray_dirs[pix * 3 + 0];
        dcy = p.ray_dirs[pix * 3 + 1];
        dcz = p.ray_dirs[pix * 3 + 2];
        m = p.ray_scale[pix];
    } else {
        dcx = fmaf(static_cast<float>(px), in.x, in.y);
        dcy = fmaf(static_cast<float>(py), in.z, in.w);
        dcz = 1.0f;
        m = sqrtf(fmaf(dcx, dcx, fmaf(dcy, dcy, 1.0f)));
    }
    const float inv_m = __frcp_rn(m);   // == 1.0f / m (both correctly rounded), fewer instructions
    TraceCounters ctr;
    float z = dmax;

    // ---- K2: links in their local frames (numba_backend.py:190-208) ----
    // Lanes load 32 links' pixel rects at once (one 8 B record each), a ballot
    // keeps the links whose rect overlaps this tile, and only those are visited
    // (in link order); inside, lanes outside the rect sit the trace out.
    const LinkRec* links = p.links + static_cast<int64_t>(view) * p.B;
    const int2* rects = p.rects + static_cast<int64_t>(view) * p.B;
    const int tx0 = static_cast<int>(tx) * kTileW, ty0 = static_cast<int>(ty) * kTileH;
    for (int base = 0; base < nlinks; base += 32) {
        int2 rr = make_int2(0, 0);
        bool ov = false;
        if (base + lane < nlinks) {
            rr = rects[base + lane];
            const int x0 = static_cast<int16_t>(rr.x & 0xffff), x1 = rr.x >> 16;
            const int y0 = static_cast<int16_t>(rr.y & 0xffff), y1 = rr.y >> 16;
            ov = !(x1 < tx0 || x0 >= tx0 + kTileW || y1 < ty0 || y0 >= ty0 + kTileH);
        }
        unsigned todo = __ballot_sync(0xffffffffu, ov);
        while (todo) {
            const int j = __ffs(todo) - 1;
            todo &= todo - 1;
            const int rx = __shfl_sync(0xffffffffu, rr.x, j), ry = __shfl_sync(0xffffffffu, rr.y, j);
            const int x0 = static_cast<int16_t>(rx & 0xffff), x1 = rx >> 16;
            const int y0 = static_cast<int16_t>(ry & 0xffff), y1 = ry >> 16;
            const bool want = active && px >= x0 && px <= x1 && py >= y0 && py <= y1;
            if (!__any_sync(0xffffffffu, want)) continue;
            if (want) {
                const LinkRec& L = links[base + j];
                const float4 m0 = *reinterpret_cast<const float4*>(&L.m[0]);
                const float4 m1 = *reinterpret_cast<const float4*>(&L.m[4]);
                const float4 m2 = *reinterpret_cast<const float4*>(&L.m[8]);  // m8 o0 o1 o2
                const float ldx = m0.x * dcx + m0.y * dcy + m0.z * dcz;
                const float ldy = m0.w * dcx + m1.x * dcy + m1.y * dcz;
                const float ldz = m1.z * dcx + m1.w * dcy + m2.x * dcz;
                const float bound = p.early_termination ? z : dmax;
                const unsigned int before = ctr.nodes;
                const float tt = trace<COUNT>(p.nodes, p.tri_tex, L.root, m2.y, m2.z, m2.w, ldx, ldy, ldz,
                                              bound * inv_m, stack, ctr, p.n_nodes, p.n_tris);
                if (COUNT) {
                    ctr.link_nodes += ctr.nodes - before;
                    ++ctr.link_traces;
                }
                const float cand = m * tt;
                if (cand < z) z = cand;
            }
        }
    }

    // ---- K1: terrain in the world frame (numba_backend.py:209-218) ----
    if (p.terrain_root >= 0 && active) {
        const float4 r0 = *reinterpret_cast<const float4*>(&V.r[0]);  // r0..r3
        const float4 r1 = *reinterpret_cast<const float4*>(&V.r[4]);  // r4..r7
        const float4 r2 = *reinterpret_cast<const float4*>(&V.r[8]);  // r8, o0, o1, o2
        const float wdx = r0.x * dcx + r0.y * dcy + r0.z * dcz;
        const float wdy = r0.w * dcx + r1.x * dcy + r1.y * dcz;
        const float wdz = r1.z * dcx + r1.w * dcy + r2.x * dcz;
        const float bound = p.early_termination ? z : dmax;
        // the prologue's entry node of this tile (a node every ray of the tile reaches first)
        const uint32_t tslot = view * static_cast<uint32_t>(p.tiles_per_view) + ty * static_cast<uint32_t>(p.tiles_x) + tx;
        MDRT_CHECK(tslot < static_cast<uint32_t>(p.N * p.C * p.tiles_per_view), "tile entry slot %u", tslot);
        const int32_t troot = p.tile_entry ? p.tile_entry[tslot] : p.terrain_root;
#ifdef MDRT_NO_OCTANT
        const float tt = trace<COUNT>(p.nodes, p.tri_tex, troot, r2.y, r2.z, r2.w, wdx, wdy, wdz,
                                      bound * inv_m, stack, ctr, p.n_nodes, p.n_tris);
#else
        const float tt = trace_oct<COUNT>(p.nodes, p.tri_tex, troot, r2.y, r2.z, r2.w, wdx, wdy, wdz,
                                          bound * inv_m, stack, ctr, p.n_nodes, p.n_tris);
#endif
        const float cand = m * tt;
        if (cand < z) z = cand;
    }

    if (COUNT) {
        unsigned int cv[4] = {ctr.nodes, ctr.tris, ctr.link_nodes, ctr.link_traces};
        for (int i = 0; i < 4; ++i) {
            for (int off = 16; off > 0; off >>= 1) cv[i] += __shfl_xor_sync(0xffffffffu, cv[i], off);
            if (lane == 0 && (i < 2 || p.count_detail))
                atomicAdd(p.counters + i, static_cast<unsigned long long>(cv[i]));
        }
    }

    // ---- K3: fused epilogue ----
    float val = z;
    if (p.sensor) {
        // a few lanes hash the tile's rows of the uniform and of the normal stream;
        // everyone picks its row's prefixes by shuffle
        // (lanes 0..kTileH-1: uniform stream rows, kTileH..2*kTileH-1: normal stream rows).
        // counter_mix of the row and column counters comes from a 512-entry table in
        // the kernel parameters (constant bank) instead of one mix64 each.
        const int hl = lane % (2 * kTileH);
        const uint32_t rrow = ty * kTileH + hl % kTileH;
        const unsigned long long rowh = mix64((hl >= kTileH ? V.hn : V.hu) ^
                                              (rrow < 512 ? p.cmix[rrow] : counter_mix(rrow)));
        const unsigned long long ru = __shfl_sync(0xffffffffu, rowh, lane / kTileW);
        const unsigned long long rn = __shfl_sync(0xffffffffu, rowh, kTileH + lane / kTileW);
        const unsigned long long cx = px < 512 ? p.cmix[px] : counter_mix(static_cast<unsigned long long>(px));
        val = sensor_apply_cx(z, ru, rn, cx, p.noise_scale, p.drop_k, p.fill[c], p.dmax64[c]);
    }
    if (active) {
        // pixel index in 32 bits (the API bounds N*C*H*W below 2^31); view = e * C + c
        const uint32_t o = (view * static_cast<uint32_t>(p.H) + static_cast<uint32_t>(py)) * static_cast<uint32_t>(p.W) +
                           static_cast<uint32_t>(px);
        if (p.out_clean) st_stream(p.out_clean + o, z);
        MDRT_CHECK(o < static_cast<uint64_t>(p.frame), "pixel index %u", o);
        if (p.ring) {
            // ring traffic streams past L1/L2 (evict-first) so it does not
            // displace BVH records; a zero-lag read is the value just written
            const int64_t frame = p.frame;   // N*C*H*W
            const int wslot = V.write_slot;   // the prologue's copy: no per-tile state load
            st_stream(p.ring + static_cast<int64_t>(wslot) * frame + o, val);
            const int rs = V.read_slot;
            MDRT_CHECK(wslot >= 0 && wslot < p.ring_slots && rs < p.ring_slots, "ring slots write %d read %d of %d",
                       wslot, rs, p.ring_slots);
            if (rs >= 0 && rs != wslot) val = __ldcs(p.ring + static_cast<int64_t>(rs) * frame + o);
        }
        if (p.rsm) {
            // random side masking of the observation (perception.py:183-202)
            const int k = V.rsm_k;
            if (k > 0 && (px < k || px >= p.W - k)) {
                const unsigned long long h = absorb(absorb(V.hr, static_cast<unsigned long long>(py)),
                                                    static_cast<unsigned long long>(px));
                val = static_cast<float>(__dadd_rn(p.rsm_low, __dmul_rn(p.rsm_high[c] - p.rsm_low, unit53(h))));
            }
        }
        if (p.out) st_stream(p.out + o, val);
    }
    if (p.ds_out) {
        // block-minimum downsample of the observation (sensor.py:85-100): lanes of
        // the same f x f block combine by warp reduction, one atomicMin per block
        // and warp (positive floats order like their bit patterns).
        const int f = p.ds_factor;
        const long long key = active ? (static_cast<long long>(view) * p.ds_h + py / f) * p.ds_w + px / f
                                     : -1LL - lane;
        MDRT_CHECK(!active || key < static_cast<long long>(p.N) * p.C * p.ds_h * p.ds_w, "ds index %lld", key);
        const unsigned grp = __match_any_sync(0xffffffffu, key);
        const unsigned mn = __reduce_min_sync(grp, __float_as_uint(val));
        if (active && lane == __ffs(grp) - 1) atomicMin(p.ds_out + key, mn);
    }
}

// Persistent warps: each warp pulls 8x4 tiles from a global counter until the
// launch's tiles are exhausted (no block-tail idling, Aila & Laine style).
#ifndef MDRT_MINB
#define MDRT_MINB 9
#endif
#ifndef MDRT_GRAB
#define MDRT_GRAB 1
#endif
#ifdef MDRT_TIMING
// diagnostic build (tools/tile_times.py): per-tile start/end global timer
__device__ unsigned long long g_tile_t0[1 << 22];
__device__ unsigned long long g_tile_t1[1 << 22];
extern "C" void mdrt_debug_tile_times(unsigned long long* t0, unsigned long long* t1, int n) {
    cudaMemcpyFromSymbol(t0, g_tile_t0, sizeof(unsigned long long) * n);
    cudaMemcpyFromSymbol(t1, g_tile_t1, sizeof(unsigned long long) * n);
}
#endif
template <bool COUNT, int TW>
static __global__ void __launch_bounds__(kBlock, MDRT_MINB) render_kernel(RenderParams p) {
    // Traversal stack in local memory: it is cached in L1 like the node
    // records, and with no shared memory reserved the whole 256 KB of the
    // SM's L1/shared array serves as data cache (a 24 KB/block shared stack
    // left ~40 KB of L1 at 9 blocks/SM and ran 4 % slower).
#ifdef MDRT_SHARED_STACK
    __shared__ int2 s_stack[kStack * kBlock];
    int2* stack = s_stack + threadIdx.x;
#else
    int2 l_stack[kStack];
    int2* stack = l_stack;
#endif
    const int lane = threadIdx.x & 31;
    const uint32_t total = static_cast<uint32_t>(p.N) * p.C * p.tiles_per_view;
    // Work order (one render_tile call site keeps the kernel's code small):
    // (0) with SM-local chunks, this SM's contiguous chunk of tiles, so
    // consecutive tiles of the same views stay on one SM and reuse node records
    // from its L1; (1) the shared pool (all tiles when there are no chunks);
    // (2) stealing what is left in other chunks (slow or absent SMs), lanes
    // probing 32 counters at once.
    const uint32_t nc = static_cast<uint32_t>(p.chunks);
    const uint32_t pool_lo = nc ? p.local_tiles : 0u;
    uint32_t own = 0;
    if (nc) {
        uint32_t smid;
        asm("mov.u32 %0, %%smid;" : "=r"(smid));
        own = smid % nc;
    }
    auto lo_of = [&](uint32_t j) {
        return static_cast<uint32_t>(static_cast<unsigned long long>(p.local_tiles) * j / nc);
    };
    uint32_t phase = nc ? 0u : 1u, base = 0;
#if MDRT_GRAB > 1 && defined(MDRT_GRAB_REG)
    // shared-pool tiles are taken MDRT_GRAB at a time (aligned groups); only the
    // last tile index stays live across a tile, the group end is recomputed
    uint32_t last = 0xffffffffu;
#elif MDRT_GRAB > 1
    // shared-pool tiles are taken MDRT_GRAB at a time; the batch's next/end
    // live in shared memory so nothing stays in registers across a tile
    __shared__ uint32_t s_batch[kBlock / 32][2];
    volatile uint32_t* sb = s_batch[threadIdx.x >> 5];
    sb[0] = 0;
    sb[1] = 0;
#endif
    while (true) {
        uint32_t gw = 0xffffffffu;
#if MDRT_GRAB > 1 && defined(MDRT_GRAB_REG)
        {
            const uint32_t nxt = last + 1;
            if (phase == 1 && ((nxt - pool_lo) & (MDRT_GRAB - 1)) != 0 && nxt < total) gw = nxt;
        }
        if (gw == 0xffffffffu)
#elif MDRT_GRAB > 1
        {
            const uint32_t nxt = sb[0];
            if (nxt < sb[1]) {
                sb[0] = nxt + 1;
                gw = nxt;
            }
        }
        if (gw == 0xffffffffu)
#endif
        while (phase < 3) {
            uint32_t ctr_idx, lo, size;
            if (phase == 0) {
                ctr_idx = own;
                lo = lo_of(own);
                size = lo_of(own + 1) - lo;
            } else if (phase == 1) {
                ctr_idx = nc;
                lo = pool_lo;
                size = total - pool_lo;
            } else {
                const uint32_t k = base + lane;
                const bool avail = k < nc &&
                    *reinterpret_cast<volatile unsigned int*>(p.tile_counter + k) < lo_of(k + 1) - lo_of(k);
                const unsigned b = __ballot_sync(0xffffffffu, avail);
                if (!b) {
                    base += 32;
                    if (base >= nc) phase = 3;
                    continue;
                }
                ctr_idx = base + __ffs(b) - 1;
                lo = lo_of(ctr_idx);
                size = lo_of(ctr_idx + 1) - lo;
            }
            uint32_t t = 0;
#if MDRT_GRAB > 1
            const uint32_t g = phase == 1 ? MDRT_GRAB : 1u;
#else
            const uint32_t g = 1u;
#endif
            if (lane == 0) t = atomicAdd(p.tile_counter + ctr_idx, g);
            t = __shfl_sync(0xffffffffu, t, 0);
            if (t < size) {
                gw = lo + t;
#if MDRT_GRAB > 1 && !defined(MDRT_GRAB_REG)
                sb[0] = gw + 1;
                sb[1] = lo + min(t + g, size);
#endif
                break;
            }
            phase = (phase == 1 && nc == 0) ? 3u : (phase < 2 ? phase + 1 : phase);
        }
        if (gw == 0xffffffffu) break;
#if MDRT_GRAB > 1 && defined(MDRT_GRAB_REG)
        last = gw;
#endif
#ifdef MDRT_TIMING
        unsigned long long t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
#endif
        render_tile<COUNT, TW>(p, gw, lane, stack);
#ifdef MDRT_TIMING
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (lane == 0 && gw < (1u << 22)) {
            g_tile_t0[gw] = t0;
            g_tile_t1[gw] = t1;
        }
#endif
    }
}

// ---------------------------------------------------------------------------
// standalone sensor-stage operators
// ---------------------------------------------------------------------------
static __global__ void noise_kernel(NoiseParams p) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t total = static_cast<int64_t>(p.N) * p.C * p.H * p.W;
    if (i >= total) return;
    const int x = static_cast<int>(i % p.W);
    const int64_t r = i / p.W;
    const int y = static_cast<int>(r % p.H);
    const int64_t r2 = r / p.H;
    const int c = static_cast<int>(r2 % p.C);
    const int64_t e = r2 / p.C;
    const unsigned long long genv = static_cast<unsigned long long>(p.env_offset + e);
    const unsigned long long ru =
        absorb(absorb(absorb(p.hu_step, genv), static_cast<unsigned long long>(c)), static_cast<unsigned long long>(y));
    const unsigned long long rn =
        absorb(absorb(absorb(p.hn_step, genv), static_cast<unsigned long long>(c)), static_cast<unsigned long long>(y));
    p.out[i] = sensor_apply(p.in[i], ru, rn, static_cast<unsigned long long>(x), p.noise_scale, p.drop_k,
                            p.fill[c], p.dmax[c]);
}

static __global__ void rsm_kernel(RsmParams p) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t total = static_cast<int64_t>(p.N) * p.C * p.H * p.W;
    if (i >= total) return;
    const int x = static_cast<int>(i % p.W);
    const int64_t r = i / p.W;
    const int y = static_cast<int>(r % p.H);
    const int64_t ec = r / p.H;
    const int c = static_cast<int>(ec % p.C);
    const int64_t e = ec / p.C;
    const int k = p.k[min(max(p.modes[ec], 0), 2)];
    float v = p.in[i];
    if (k > 0 && (x < k || x >= p.W - k)) {
        const unsigned long long h =
            absorb(absorb(absorb(absorb(p.hr_step, static_cast<unsigned long long>(p.env_offset + e)),
                                 static_cast<unsigned long long>(c)),
                          static_cast<unsigned long long>(y)),
                   static_cast<unsigned long long>(x));
        v = static_cast<float>(__dadd_rn(p.low, __dmul_rn(p.high[c] - p.low, unit53(h))));
    }
    p.out[i] = v;
}

static __global__ void gather_kernel(GatherParams p) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= p.N * p.per_env) return;
    const int64_t e = i / p.per_env;
    const int s = p.slot[e];
    p.out[i] = p.frames[s][i];
}

static __global__ void select_kernel(SelectParams p) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= p.N) return;
    const double target = p.now - p.delays[e];
    int lo = 0, hi = p.K;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (target < p.times[mid]) hi = mid;
        else lo = mid + 1;
    }
    const int k = lo - 1 < 0 ? 0 : lo - 1;
    p.slot[e] = p.order[k];
}

static __global__ void downsample_kernel(DownsampleParams p) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int ho = p.H / p.f, wo = p.W / p.f;
    if (i >= p.planes * ho * wo) return;
    const int bx = static_cast<int>(i % wo);
    const int64_t r = i / wo;
    const int by = static_cast<int>(r % ho);
    const int64_t plane = r / ho;
    const float* src = p.in + (plane * p.H + static_cast<int64_t>(by) * p.f) * p.W + static_cast<int64_t>(bx) * p.f;
    float mn = src[0];
    for (int dy = 0; dy < p.f; ++dy)
        for (int dx = 0; dx < p.f; ++dx) {
            const float v = src[static_cast<int64_t>(dy) * p.W + dx];
            mn = v < mn ? v : mn;
        }
    p.out[i] = mn;
}

// depth_to_u8 (frameio.py depth_to_u8): round(255 * (1 - clip(d / d_max, 0, 1))) in f64,
// round-half-even like np.round; 4 pixels per thread (16 B in, 4 B out).
__device__ __forceinline__ uint8_t gray_of(float d, double dmax) {
    double f = __ddiv_rn(static_cast<double>(d), dmax);
    f = f < 0.0 ? 0.0 : (f > 1.0 ? 1.0 : f);
    return static_cast<uint8_t>(rint(__dmul_rn(255.0, __dadd_rn(1.0, -f))));
}

static __global__ void depth_u8_kernel(const float* __restrict__ in, uint8_t* __restrict__ out, int64_t n,
                                       double dmax) {
    const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t i = q * 4;
    if (i + 4 <= n) {
        const float4 v = *reinterpret_cast<const float4*>(in + i);
        uchar4 o;
        o.x = gray_of(v.x, dmax);
        o.y = gray_of(v.y, dmax);
        o.z = gray_of(v.z, dmax);
        o.w = gray_of(v.w, dmax);
        *reinterpret_cast<uchar4*>(out + i) = o;
    } else {
        for (int64_t k = i; k < n; ++k) out[k] = gray_of(in[k], dmax);
    }
}

// query_bvh: one thread per ray through one packed tree, closest hit + face
static __global__ void __launch_bounds__(128) query_kernel(QueryParams p) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= p.n) return;
    int2 stack[kStack];
    TraceCounters ctr;
    Traversal<false, true> tv;
    tv.init(p.root, p.origins[3 * i], p.origins[3 * i + 1], p.origins[3 * i + 2], p.dirs[3 * i], p.dirs[3 * i + 1],
            p.dirs[3 * i + 2], p.t_max, stack);
    MDRT_SET_LIMITS(tv, p.n_nodes, p.n_tris);
    while (!tv.round(p.nodes, p.tris, ctr)) {
    }
    p.t_out[i] = tv.result();
    p.face_out[i] = tv.hit ? tv.face : -1;
}

// read-bandwidth probe (roofline denominator of the L2-resident traversal):
// grid-stride 32 B loads that bypass L1 (ld.global.cg: served by L2 when the
// buffer is L2-resident), one partial sum per block. Launch shape from a sweep
// (tools/micro/l2_probe_sweep.cu: 8-64 MiB, 4/8/16 blocks per SM, 16/32 B loads,
// 1/4/8 in flight): 4 blocks of 256 threads per SM and one load in flight per
// thread read fastest (17.7 TB/s at 32 MiB, 18.9 TB/s at 64 MiB).
__device__ __forceinline__ void ldcg256(const float4* p, float4& a, float4& b) {
    asm volatile("ld.global.cg.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
                 : "l"(p));
}
static __global__ void __launch_bounds__(256) probe_read_kernel(const float4* __restrict__ buf, int64_t n16,
                                                                int iters, float* sink) {
    float acc = 0.f;
    const int64_t n32 = n16 / 2;                       // 32 B items
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int it = 0; it < iters; ++it) {
        for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n32; i += stride) {
            float4 a, b;
            ldcg256(buf + 2 * i, a, b);
            acc += ((a.x + a.y) + (a.z + a.w)) + ((b.x + b.y) + (b.z + b.w));
        }
    }
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    __shared__ float s[8];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.f;
        for (int w = 0; w < 8; ++w) t += s[w];
        sink[blockIdx.x] = t;
    }
}

// Advance the device step state to step k = next_step (single thread; first
// node of a captured step). Mirrors FrameBuffer._reserve + push (sensor.py:122-131)
// and the sensor stream prefix absorb(absorb(key, 0|1), k) (rng.py:71-75).
static __global__ void advance_kernel(StepState* st) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const long long k = st->next_step;
    st->now = st->t0 + static_cast<double>(k) * st->dt;
    st->hu_step = absorb(absorb(st->key, 0ULL), static_cast<unsigned long long>(k));
    st->hn_step = absorb(absorb(st->key, 1ULL), static_cast<unsigned long long>(k));
    st->hr_step = absorb(st->rsm_key, static_cast<unsigned long long>(k));
    if (st->ring_slots > 0) {
        int slot;
        if (st->ring_count < st->ring_slots) {
            slot = 0;   // lowest slot not in use
            while (true) {
                bool used = false;
                for (int i = 0; i < st->ring_count; ++i) used |= st->order[i] == slot;
                if (!used) break;
                ++slot;
            }
            ++st->ring_count;
        } else {
            slot = st->order[0];
            for (int i = 1; i < st->ring_count; ++i) {
                st->order[i - 1] = st->order[i];
                st->times[i - 1] = st->times[i];
            }
        }
        st->order[st->ring_count - 1] = slot;
        st->times[st->ring_count - 1] = st->now;
        st->write_slot = slot;
    }
    st->next_step = k + 1;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static unsigned grid_for(int64_t threads, int block) {
    return static_cast<unsigned>((threads + block - 1) / block);
}

void launch_prologue(const PrologueParams& p, int64_t views, cudaStream_t s) {
    prologue_kernel<<<grid_for(views * 32, 128), 128, 0, s>>>(p);
}

void launch_entry(const EntryParams& p, cudaStream_t s) {
    entry_kernel<<<grid_for(p.views_count * p.tiles_per_view, 128), 128, 0, s>>>(p);
}

int render_tile_width(int W) {
    // 4 x 8 tiles for narrow images (64-wide: +0.7 % at configs 2 and 3), 8 x 4
    // otherwise (160- and 240-wide: +0.4..1.3 %); MDRT_TILE_W (4 or 8) overrides
    static int env_tw = -1;
    if (env_tw < 0) {
        const char* t = std::getenv("MDRT_TILE_W");
        env_tw = t ? std::atoi(t) : 0;
    }
    if (env_tw == 4 || env_tw == 8) return env_tw;
    return W <= 96 ? 4 : 8;
}

template <int TW>
static void launch_render_tw(const RenderParams& p, int64_t warps, bool count, int64_t geometry_bytes,
                             cudaStream_t s) {
    // persistent grid: as many blocks as can be co-resident (capped by the work)
    static int blocks_per_sm[2] = {0, 0};
    static int sms = 0;
    static int l2_bytes = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&l2_bytes, cudaDevAttrL2CacheSize, dev);
        if (const char* cv = std::getenv("MDRT_CARVEOUT")) {   // experiment: shared-memory carveout %
            cudaFuncSetAttribute(render_kernel<false, TW>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 std::atoi(cv));
            cudaFuncSetAttribute(render_kernel<true, TW>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 std::atoi(cv));
        }
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm[0], render_kernel<false, TW>, kBlock, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm[1], render_kernel<true, TW>, kBlock, 0);
    }
    const int64_t need = (warps * 32 + kBlock - 1) / kBlock;
    const int64_t grid = std::min<int64_t>(need, static_cast<int64_t>(sms) * std::max(1, blocks_per_sm[count]));
    RenderParams q = p;
    {
        // SM-local chunks (95 % of the tiles, the rest dynamic) when the BVH
        // exceeds L2 and every SM gets several waves of warps. Measured: +1.7 %
        // at config 5 (270 MB BVH), -1.7 % at config 2 (21 MB, L2-resident,
        // where all SMs sharing the same views keeps L2 hot). MDRT_LOCAL_FRAC
        // overrides the fraction (0 = off).
        static double env_frac = -2.0;
        if (env_frac < -1.0) {
            const char* f = std::getenv("MDRT_LOCAL_FRAC");
            env_frac = f ? std::atof(f) : -1.0;
        }
        const double frac = env_frac >= 0.0 ? env_frac : (geometry_bytes > l2_bytes ? 0.95 : 0.0);
        const int64_t resident = static_cast<int64_t>(sms) * std::max(1, blocks_per_sm[count]) * (kBlock / 32);
        if (frac > 0.0 && sms < kTileCounters && warps >= 4 * resident) {
            q.chunks = sms;
            q.local_tiles = static_cast<uint32_t>(static_cast<double>(warps) * std::min(frac, 1.0));
        } else {
            q.chunks = 0;
            q.local_tiles = 0;
        }
        // Tile order: tile-row-major over all views unless the tiles are
        // scheduled SM-locally (there view-major chunks keep an SM on the same
        // envs' geometry). The last ~0.1 ms of a view-major launch is a few
        // horizon-row tiles costing ~20x the mean (tools/tile_times.py); taking
        // every view's top rows first ends the launch on cheap rows: config 2
        // +3.0 %, paper +1.1 %, config 3 +-0 (config 5 view-major: row-major
        // would cost 6 %). MDRT_TILE_ORDER=view|row overrides.
        static int env_order = -2;
        if (env_order == -2) {
            const char* o = std::getenv("MDRT_TILE_ORDER");
            env_order = !o ? -1 : (std::strcmp(o, "row") == 0 ? 1 : 0);
        }
        q.row_order = env_order >= 0 ? env_order : (q.chunks == 0 ? 1 : 0);
        q.order_d1 = q.row_order ? q.row_tiles : static_cast<uint32_t>(q.tiles_per_view);
        q.order_m1 = q.row_order ? q.m_row_tiles : q.m_tiles_per_view;
    }
    // Experiment (MDRT_L2_PERSIST=1, BVH larger than L2): mark the node records as
    // persisting in L2 for this launch (access-policy window launch attribute), so
    // triangle and I/O traffic cannot evict them.
    static int persist = -1;
    if (persist < 0) {
        const char* e = std::getenv("MDRT_L2_PERSIST");
        persist = e && std::atoi(e) > 0;
        if (persist) {
            int dev = 0, max_persist = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
            cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, static_cast<size_t>(max_persist));
        }
    }
    if (persist && geometry_bytes > l2_bytes) {
        int dev = 0, max_win = 0;
        size_t limit = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, dev);
        cudaDeviceGetLimit(&limit, cudaLimitPersistingL2CacheSize);
        const size_t node_bytes = static_cast<size_t>(p.n_nodes) * 64;
        const size_t win = std::min(node_bytes, static_cast<size_t>(max_win));
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[0].val.accessPolicyWindow.base_ptr = const_cast<float4*>(p.nodes);
        attr[0].val.accessPolicyWindow.num_bytes = win;
        attr[0].val.accessPolicyWindow.hitRatio = win > 0 ? std::min(1.0f, static_cast<float>(limit) / win) : 0.f;
        attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(static_cast<unsigned>(grid));
        cfg.blockDim = dim3(kBlock);
        cfg.stream = s;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (count)
            cudaLaunchKernelEx(&cfg, render_kernel<true, TW>, q);
        else
            cudaLaunchKernelEx(&cfg, render_kernel<false, TW>, q);
        return;
    }
    if (count)
        render_kernel<true, TW><<<static_cast<unsigned>(grid), kBlock, 0, s>>>(q);
    else
        render_kernel<false, TW><<<static_cast<unsigned>(grid), kBlock, 0, s>>>(q);
}

void launch_render(const RenderParams& p, int64_t warps, bool count, int64_t geometry_bytes, cudaStream_t s) {
    if (p.tile_w == 4)
        launch_render_tw<4>(p, warps, count, geometry_bytes, s);
    else
        launch_render_tw<8>(p, warps, count, geometry_bytes, s);
}

void launch_noise(const NoiseParams& p, int64_t total, cudaStream_t s) {
    noise_kernel<<<grid_for(total, 256), 256, 0, s>>>(p);
}

void launch_gather(const GatherParams& p, int64_t total, cudaStream_t s) {
    gather_kernel<<<grid_for(total, 256), 256, 0, s>>>(p);
}

void launch_select(const SelectParams& p, int64_t n, cudaStream_t s) {
    select_kernel<<<grid_for(n, 256), 256, 0, s>>>(p);
}

void launch_probe_read(const float4* buf, int64_t n16, int iters, float* sink, cudaStream_t s) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    probe_read_kernel<<<sms * 4, 256, 0, s>>>(buf, n16, iters, sink);
}

void launch_advance(StepState* st, cudaStream_t s) { advance_kernel<<<1, 32, 0, s>>>(st); }

void launch_rsm(const RsmParams& p, int64_t total, cudaStream_t s) {
    rsm_kernel<<<grid_for(total, 256), 256, 0, s>>>(p);
}

void launch_downsample(const DownsampleParams& p, int64_t total, cudaStream_t s) {
    downsample_kernel<<<grid_for(total, 256), 256, 0, s>>>(p);
}

void launch_query(const QueryParams& p, cudaStream_t s) {
    query_kernel<<<grid_for(p.n, 128), 128, 0, s>>>(p);
}

void launch_depth_u8(const float* in, uint8_t* out, int64_t n, double dmax, cudaStream_t s) {
    depth_u8_kernel<<<grid_for((n + 3) / 4, 256), 256, 0, s>>>(in, out, n, dmax);
}

}  // namespace mdrt
