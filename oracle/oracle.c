/*
 * oracle.c -- CPU restatement of the reference depth path. TEST INFRASTRUCTURE ONLY.
 *
 * This file is the parity checker for the B200 renderer. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it; the product path (paper_2602_03002_b200) never does.
 *
 * It restates, in plain C with IEEE double arithmetic (built with
 * -ffp-contract=off so no FMA contraction changes rounding), the algorithm of
 * the reference package `multidepth` (paths relative to
 * /root/reference/pkg/src/multidepth):
 *
 *   orc_build_bvh        bvh.py:68-136            median split, stable sort, leaf <= 4
 *   orc_render           kernels/numba_backend.py:155-219  (_render_kernel)
 *     rotate_q           kernels/numba_backend.py:25-34    (_rotate)
 *     tri_t              kernels/numba_backend.py:37-69    (_tri_t, Moller-Trumbore)
 *     slab_hit           kernels/numba_backend.py:72-121   (_slab_hit)
 *     closest_hit        kernels/numba_backend.py:124-152  (_closest_hit)
 *   orc_mix64/absorb     rng.py:30-58
 *   orc_stream_key       rng.py:61-68
 *   orc_uniform/normal   rng.py:71-99
 *   orc_noise_dropout    sensor.py:55-82           (apply_noise_dropout)
 *   orc_frame_select     sensor.py:133-150         (FrameBuffer.fetch_delayed[_batch])
 *   orc_downsample_min   sensor.py:85-100          (downsample_min)
 *   orc_rsm_apply        perception.py:169-202     (rsm_apply, random side masking)
 *
 * Parity of this restatement against the live reference is pinned by
 * tests/golden/make_golden.py (run where /root/reference exists) and
 * tests/test_oracle_golden.py (runs everywhere against the committed vectors).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define RAY_EPSILON 1e-6
#define DET_EPSILON 1e-12
#define STACK_DEPTH 128

/* ------------------------------------------------------------------------- */
/* BVH build: bvh.py:68-136                                                   */
/* ------------------------------------------------------------------------- */

typedef struct {
    const double *key;
    int64_t *sel;
} sort_ctx;

/* Stable sort of sel[0:n] by key[sel[i]] (merge sort; equals numpy's
 * argsort(kind="stable") applied to the current order). */
static void stable_sort_by_key(int64_t *sel, int64_t n, const double *key, int64_t *tmp) {
    if (n < 2) return;
    int64_t mid = n / 2;
    stable_sort_by_key(sel, mid, key, tmp);
    stable_sort_by_key(sel + mid, n - mid, key, tmp);
    int64_t i = 0, j = mid, k = 0;
    while (i < mid && j < n) {
        /* take from the right run only when strictly smaller -> stable */
        if (key[sel[j]] < key[sel[i]]) tmp[k++] = sel[j++];
        else tmp[k++] = sel[i++];
    }
    while (i < mid) tmp[k++] = sel[i++];
    while (j < n) tmp[k++] = sel[j++];
    memcpy(sel, tmp, (size_t)n * sizeof(int64_t));
}

/* tris: (F,3,3) f64. Outputs sized for 2F-1 nodes. Returns node count M.
 * keys_scratch: F*3 doubles (centroid per axis, axis-major). */
int64_t orc_build_bvh(const double *tris, int64_t F, int leaf_size,
                      double *node_min, double *node_max,
                      int32_t *left, int32_t *right, int32_t *start, int32_t *count,
                      int64_t *tri_index) {
    if (F <= 0 || leaf_size < 1) return -1;
    double *tmin = (double *)malloc(sizeof(double) * 3 * F);
    double *tmax = (double *)malloc(sizeof(double) * 3 * F);
    double *cen = (double *)malloc(sizeof(double) * 3 * F); /* axis-major */
    int64_t *tmp = (int64_t *)malloc(sizeof(int64_t) * F);
    int64_t *stk = (int64_t *)malloc(sizeof(int64_t) * 3 * (2 * F + 2));
    for (int64_t f = 0; f < F; ++f) {
        for (int a = 0; a < 3; ++a) {
            double x0 = tris[f * 9 + 0 * 3 + a], x1 = tris[f * 9 + 1 * 3 + a], x2 = tris[f * 9 + 2 * 3 + a];
            double lo = x0 < x1 ? x0 : x1; lo = lo < x2 ? lo : x2;
            double hi = x0 > x1 ? x0 : x1; hi = hi > x2 ? hi : x2;
            tmin[f * 3 + a] = lo;
            tmax[f * 3 + a] = hi;
            cen[a * F + f] = 0.5 * (lo + hi);
        }
        tri_index[f] = f;
    }
    int64_t M = 0;
#define NEW_NODE(LO, HI)                                                        \
    do {                                                                        \
        double mn[3] = {INFINITY, INFINITY, INFINITY};                          \
        double mx[3] = {-INFINITY, -INFINITY, -INFINITY};                       \
        for (int64_t q = (LO); q < (HI); ++q) {                                 \
            int64_t t = tri_index[q];                                           \
            for (int a = 0; a < 3; ++a) {                                       \
                if (tmin[t * 3 + a] < mn[a]) mn[a] = tmin[t * 3 + a];           \
                if (tmax[t * 3 + a] > mx[a]) mx[a] = tmax[t * 3 + a];           \
            }                                                                   \
        }                                                                       \
        for (int a = 0; a < 3; ++a) { node_min[M * 3 + a] = mn[a]; node_max[M * 3 + a] = mx[a]; } \
        left[M] = -1; right[M] = -1; start[M] = 0; count[M] = 0;                \
        ++M;                                                                    \
    } while (0)

    NEW_NODE(0, F);
    int64_t sp = 0;
    stk[0] = 0; stk[1] = 0; stk[2] = F; sp = 1;
    while (sp > 0) {
        --sp;
        int64_t node = stk[sp * 3 + 0], lo = stk[sp * 3 + 1], hi = stk[sp * 3 + 2];
        int64_t n = hi - lo;
        if (n <= leaf_size) {
            start[node] = (int32_t)lo;
            count[node] = (int32_t)n;
            continue;
        }
        int axis = 0;
        double best = node_max[node * 3 + 0] - node_min[node * 3 + 0];
        for (int a = 1; a < 3; ++a) {
            double e = node_max[node * 3 + a] - node_min[node * 3 + a];
            if (e > best) { best = e; axis = a; } /* np.argmax: first maximum */
        }
        stable_sort_by_key(tri_index + lo, n, cen + (int64_t)axis * F, tmp);
        int64_t mid = lo + n / 2;
        int64_t lc = M; NEW_NODE(lo, mid);
        int64_t rc = M; NEW_NODE(mid, hi);
        left[node] = (int32_t)lc;
        right[node] = (int32_t)rc;
        /* push right then left so left is processed first */
        stk[sp * 3 + 0] = rc; stk[sp * 3 + 1] = mid; stk[sp * 3 + 2] = hi; ++sp;
        stk[sp * 3 + 0] = lc; stk[sp * 3 + 1] = lo; stk[sp * 3 + 2] = mid; ++sp;
    }
#undef NEW_NODE
    free(tmin); free(tmax); free(cen); free(tmp); free(stk);
    return M;
}

/* ------------------------------------------------------------------------- */
/* Traversal: kernels/numba_backend.py:25-152                                 */
/* ------------------------------------------------------------------------- */

static inline void rotate_q(double qw, double qx, double qy, double qz,
                            double vx, double vy, double vz,
                            double *rx, double *ry, double *rz) {
    double tx = 2.0 * (qy * vz - qz * vy);
    double ty = 2.0 * (qz * vx - qx * vz);
    double tz = 2.0 * (qx * vy - qy * vx);
    *rx = vx + qw * tx + (qy * tz - qz * ty);
    *ry = vy + qw * ty + (qz * tx - qx * tz);
    *rz = vz + qw * tz + (qx * ty - qy * tx);
}

/* Barycentric margin of the triangle test: 0 (the reference's exact u in [0,1],
 * v >= 0, u + v <= 1, numba_backend.py:58-64) unless a parity diagnostic sets
 * the GPU kernel's fp32 watertightness margin (kBaryEps) to classify hit/miss
 * flips (bench.py parity block). Test infrastructure only. */
static double g_bary_eps = 0.0;
void orc_set_bary_eps(double eps) { g_bary_eps = eps; }

static inline double tri_t(const double *v0, const double *v1, const double *v2, int64_t i,
                           double ox, double oy, double oz, double dx, double dy, double dz,
                           double t_max) {
    const double *a = v0 + 3 * i, *b = v1 + 3 * i, *c = v2 + 3 * i;
    double e1x = b[0] - a[0], e1y = b[1] - a[1], e1z = b[2] - a[2];
    double e2x = c[0] - a[0], e2y = c[1] - a[1], e2z = c[2] - a[2];
    double px = dy * e2z - dz * e2y;
    double py = dz * e2x - dx * e2z;
    double pz = dx * e2y - dy * e2x;
    double det = e1x * px + e1y * py + e1z * pz;
    double miss = t_max + 1.0;
    if (det < DET_EPSILON && det > -DET_EPSILON) return miss;
    double inv_det = 1.0 / det;
    double tx = ox - a[0], ty = oy - a[1], tz = oz - a[2];
    double u = (tx * px + ty * py + tz * pz) * inv_det;
    const double be = g_bary_eps;
    if (u < -be || u > 1.0 + be) return miss;
    double qx = ty * e1z - tz * e1y;
    double qy = tz * e1x - tx * e1z;
    double qz = tx * e1y - ty * e1x;
    double v = (dx * qx + dy * qy + dz * qz) * inv_det;
    if (v < -be || u + v > 1.0 + be) return miss;
    double t = (e2x * qx + e2y * qy + e2z * qz) * inv_det;
    if (t <= RAY_EPSILON || t > t_max) return miss;
    return t;
}

static inline int slab_axis(double b0, double b1, double o, double d, double *t0, double *t1) {
    if (d == 0.0) return !(o < b0 || o > b1);
    double inv = 1.0 / d;
    double ta = (b0 - o) * inv, tb = (b1 - o) * inv;
    if (ta > tb) { double s = ta; ta = tb; tb = s; }
    if (ta > *t0) *t0 = ta;
    if (tb < *t1) *t1 = tb;
    return !(*t0 > *t1);
}

static inline int slab_hit(const double *bmin, const double *bmax,
                           double ox, double oy, double oz, double dx, double dy, double dz,
                           double bound) {
    double t0 = 0.0, t1 = bound;
    if (!slab_axis(bmin[0], bmax[0], ox, dx, &t0, &t1)) return 0;
    if (!slab_axis(bmin[1], bmax[1], oy, dy, &t0, &t1)) return 0;
    if (!slab_axis(bmin[2], bmax[2], oz, dz, &t0, &t1)) return 0;
    return 1;
}

typedef struct {
    const double *node_min, *node_max;
    const int32_t *left, *right, *start, *count;
    const double *v0, *v1, *v2;
} orc_tree;

/* counters (optional): [0] node visits, [1] triangle tests */
static inline double closest_hit(const orc_tree *g, int64_t root,
                                 double ox, double oy, double oz, double dx, double dy, double dz,
                                 double t_max, int64_t *stack, int64_t *ctr) {
    double best = t_max;
    int top = 0;
    stack[top++] = root;
    while (top > 0) {
        int64_t node = stack[--top];
        if (ctr) ctr[0]++;
        if (!slab_hit(g->node_min + 3 * node, g->node_max + 3 * node, ox, oy, oz, dx, dy, dz, best))
            continue;
        if (g->left[node] < 0) {
            int64_t s = g->start[node], e = s + g->count[node];
            for (int64_t i = s; i < e; ++i) {
                if (ctr) ctr[1]++;
                double t = tri_t(g->v0, g->v1, g->v2, i, ox, oy, oz, dx, dy, dz, best);
                if (t < best) best = t;
            }
        } else {
            stack[top++] = g->right[node];
            stack[top++] = g->left[node];
        }
    }
    return best;
}

/* Mirrors _render_kernel's argument list (numba_backend.py:156-162), with the
 * forest/terrain arrays passed flat. ray_dirs (RN,C,H,W,3), ray_scale (RN,C,H,W).
 * counters (optional, length 2) accumulate node visits / triangle tests. */
void orc_render(int64_t N, int64_t C, int64_t H, int64_t W, int64_t B, int64_t RN,
                const double *cam_pos, const double *cam_rot,
                const double *ray_dirs, const double *ray_scale,
                const double *body_pos, const double *body_rot, const int32_t *body_root,
                const double *node_min, const double *node_max,
                const int32_t *left, const int32_t *right, const int32_t *start, const int32_t *count,
                const double *tri_v0, const double *tri_v1, const double *tri_v2,
                int64_t g_nodes,
                const double *g_node_min, const double *g_node_max,
                const int32_t *g_left, const int32_t *g_right, const int32_t *g_start, const int32_t *g_count,
                const double *g_tri_v0, const double *g_tri_v1, const double *g_tri_v2,
                const double *d_max, int early_term, float *out, int threads, int64_t *counters) {
    orc_tree bodies = {node_min, node_max, left, right, start, count, tri_v0, tri_v1, tri_v2};
    orc_tree terr = {g_node_min, g_node_max, g_left, g_right, g_start, g_count, g_tri_v0, g_tri_v1, g_tri_v2};
    int has_terrain = g_nodes > 0;
    int64_t rows = N * C * H;
    int64_t c_nodes = 0, c_tris = 0;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(dynamic, 4) reduction(+ : c_nodes, c_tris)
#endif
    for (int64_t row = 0; row < rows; ++row) {
        int64_t e = row / (C * H);
        int64_t rem = row - e * (C * H);
        int64_t c = rem / H;
        int64_t y = rem - c * H;
        int64_t er = RN > 1 ? e : 0;
        int64_t stack[STACK_DEPTH];
        int64_t ctr[2] = {0, 0};
        int64_t *pc = counters ? ctr : NULL;
        double far = d_max[c];
        const double *cq = cam_rot + (e * C + c) * 4;
        const double *cp = cam_pos + (e * C + c) * 3;
        for (int64_t x = 0; x < W; ++x) {
            int64_t pix = ((er * C + c) * H + y) * W + x;
            double m = ray_scale[pix];
            double wdx, wdy, wdz;
            rotate_q(cq[0], cq[1], cq[2], cq[3], ray_dirs[pix * 3 + 0], ray_dirs[pix * 3 + 1],
                     ray_dirs[pix * 3 + 2], &wdx, &wdy, &wdz);
            double z_star = far;
            for (int64_t b = 0; b < B; ++b) {
                double bound = early_term ? z_star : far;
                double t_bound = bound / m;
                const double *bq = body_rot + (e * B + b) * 4;
                const double *bp = body_pos + (e * B + b) * 3;
                double rx = cp[0] - bp[0], ry = cp[1] - bp[1], rz = cp[2] - bp[2];
                double box, boy, boz, bdx, bdy, bdz;
                rotate_q(bq[0], -bq[1], -bq[2], -bq[3], rx, ry, rz, &box, &boy, &boz);
                rotate_q(bq[0], -bq[1], -bq[2], -bq[3], wdx, wdy, wdz, &bdx, &bdy, &bdz);
                double t = closest_hit(&bodies, body_root[b], box, boy, boz, bdx, bdy, bdz, t_bound, stack, pc);
                double cand = m * t;
                if (cand < z_star) z_star = cand;
            }
            if (has_terrain) {
                double bound = early_term ? z_star : far;
                double t_bound = bound / m;
                double t = closest_hit(&terr, 0, cp[0], cp[1], cp[2], wdx, wdy, wdz, t_bound, stack, pc);
                double cand = m * t;
                if (cand < z_star) z_star = cand;
            }
            out[((e * C + c) * H + y) * W + x] = (float)z_star;
        }
        c_nodes += ctr[0];
        c_tris += ctr[1];
    }
    if (counters) { counters[0] += c_nodes; counters[1] += c_tris; }
}

/* ------------------------------------------------------------------------- */
/* Counter-based RNG: rng.py:30-99                                            */
/* ------------------------------------------------------------------------- */

#define GOLDEN 0x9E3779B97F4A7C15ULL
#define MIX_A 0xBF58476D1CE4E5B9ULL
#define MIX_B 0x94D049BB133111EBULL
#define DOM_NORMAL_U1 0x9A4C93AED1F3B217ULL
#define DOM_NORMAL_U2 0x6E2F1D84C5A7093BULL
static const double INV_2_53 = 1.0 / 9007199254740992.0; /* 2**-53 */

uint64_t orc_mix64(uint64_t x) {
    x ^= x >> 30;
    x *= MIX_A;
    x ^= x >> 27;
    x *= MIX_B;
    x ^= x >> 31;
    return x;
}

uint64_t orc_absorb(uint64_t h, uint64_t v) { return orc_mix64(h ^ orc_mix64(v + GOLDEN)); }

/* stream name bytes (utf-8), length n */
uint64_t orc_stream_key(int64_t seed, const unsigned char *name, int64_t n) {
    uint64_t h = orc_absorb(GOLDEN, (uint64_t)seed);
    h = orc_absorb(h, (uint64_t)n);
    for (int64_t i = 0; i < n; i += 8) {
        uint64_t chunk = 0;
        for (int64_t k = 0; k < 8 && i + k < n; ++k) chunk |= (uint64_t)name[i + k] << (8 * k);
        h = orc_absorb(h, chunk);
    }
    return h;
}

static inline double unit_closed_open(uint64_t h) { return (double)(h >> 11) * INV_2_53; }
static inline double unit_open_closed(uint64_t h) { return (double)((h >> 11) + 1ULL) * INV_2_53; }

static inline double normal_from_hash(uint64_t h) {
    double u1 = unit_open_closed(orc_absorb(h, DOM_NORMAL_U1));
    double u2 = unit_closed_open(orc_absorb(h, DOM_NORMAL_U2));
    return sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
}

/* counters: (n, k) int64 row-major; writes n values */
void orc_uniform(uint64_t key, const int64_t *counters, int64_t n, int64_t k, double low, double high,
                 double *out) {
    for (int64_t i = 0; i < n; ++i) {
        uint64_t h = key;
        for (int64_t j = 0; j < k; ++j) h = orc_absorb(h, (uint64_t)counters[i * k + j]);
        out[i] = low + (high - low) * unit_closed_open(h);
    }
}

void orc_normal(uint64_t key, const int64_t *counters, int64_t n, int64_t k, double *out) {
    for (int64_t i = 0; i < n; ++i) {
        uint64_t h = key;
        for (int64_t j = 0; j < k; ++j) h = orc_absorb(h, (uint64_t)counters[i * k + j]);
        out[i] = normal_from_hash(h);
    }
}

/* apply_noise_dropout: sensor.py:55-82. depth/out (N,C,H,W) f32; d_max, fill (C,).
 * env index = env_offset + e (global env id; the reference uses arange(N)). */
void orc_noise_dropout(const float *depth, int64_t N, int64_t C, int64_t H, int64_t W,
                       int64_t env_offset, const double *d_max, const double *fill,
                       double noise_scale, double dropout_p, uint64_t key, int64_t step,
                       float *out, int threads) {
    int64_t rows = N * C * H;
    uint64_t hu = orc_absorb(orc_absorb(key, 0), (uint64_t)step);
    uint64_t hn = orc_absorb(orc_absorb(key, 1), (uint64_t)step);
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(static)
#endif
    for (int64_t row = 0; row < rows; ++row) {
        int64_t e = row / (C * H);
        int64_t rem = row - e * (C * H);
        int64_t c = rem / H;
        int64_t y = rem - c * H;
        uint64_t ru = orc_absorb(orc_absorb(orc_absorb(hu, (uint64_t)(env_offset + e)), (uint64_t)c), (uint64_t)y);
        uint64_t rn = orc_absorb(orc_absorb(orc_absorb(hn, (uint64_t)(env_offset + e)), (uint64_t)c), (uint64_t)y);
        double lo = 1e-6, hi = d_max[c];
        for (int64_t x = 0; x < W; ++x) {
            int64_t i = row * W + x;
            int drop = unit_closed_open(orc_absorb(ru, (uint64_t)x)) < dropout_p;
            double g = normal_from_hash(orc_absorb(rn, (uint64_t)x));
            double noisy = (double)depth[i] * (1.0 + noise_scale * g);
            double v = drop ? fill[c] : noisy;
            /* np.clip(a, lo, hi) == minimum(maximum(a, lo), hi) */
            v = v > lo ? v : lo;
            v = v < hi ? v : hi;
            out[i] = (float)v;
        }
    }
}

/* FrameBuffer.fetch_delayed_batch index selection (sensor.py:133-150):
 * idx_e = max(bisect_right(times, now - delay_e) - 1, 0). times: K increasing. */
void orc_frame_select(const double *times, int64_t K, double now, const double *delays, int64_t N,
                      int64_t *idx) {
    for (int64_t e = 0; e < N; ++e) {
        double target = now - delays[e];
        int64_t lo = 0, hi = K; /* bisect_right */
        while (lo < hi) {
            int64_t mid = (lo + hi) / 2;
            if (target < times[mid]) hi = mid;
            else lo = mid + 1;
        }
        int64_t k = lo - 1;
        idx[e] = k < 0 ? 0 : k;
    }
}

/* downsample_min: sensor.py:85-100, over trailing (H,W) of `planes` images. */
void orc_downsample_min(const float *in, int64_t planes, int64_t H, int64_t W, int64_t f, float *out) {
    int64_t ho = H / f, wo = W / f;
    for (int64_t p = 0; p < planes; ++p)
        for (int64_t by = 0; by < ho; ++by)
            for (int64_t bx = 0; bx < wo; ++bx) {
                float m = in[(p * H + by * f) * W + bx * f];
                for (int64_t dy = 0; dy < f; ++dy)
                    for (int64_t dx = 0; dx < f; ++dx) {
                        float v = in[(p * H + by * f + dy) * W + bx * f + dx];
                        if (v < m) m = v;
                    }
                out[(p * ho + by) * wo + bx] = m;
            }
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* rsm_apply: perception.py:169-202. Side bands of k = int(f * W) columns per
 * side (mode 0: none, 1: f_small, 2: f_large; k passed per mode) are
 * overwritten with uniform(key, step, env, cam, row, col, low, high_c) cast to
 * f32; all other pixels are copied bit-identically. env = env_offset + e. */
void orc_rsm_apply(const float *depth, int64_t N, int64_t C, int64_t H, int64_t W, const int32_t *modes,
                   const int64_t *k_for_mode, uint64_t key, int64_t step, int64_t env_offset, double low,
                   const double *high, float *out) {
    memcpy(out, depth, sizeof(float) * (size_t)(N * C * H * W));
    for (int64_t e = 0; e < N; ++e)
        for (int64_t c = 0; c < C; ++c) {
            int64_t k = k_for_mode[modes[e * C + c]];
            if (k == 0) continue;
            uint64_t hc = orc_absorb(orc_absorb(orc_absorb(key, (uint64_t)step), (uint64_t)(env_offset + e)),
                                     (uint64_t)c);
            for (int64_t y = 0; y < H; ++y) {
                uint64_t hy = orc_absorb(hc, (uint64_t)y);
                for (int64_t x = 0; x < W; ++x) {
                    if (x >= k && x < W - k) continue;
                    double u = unit_closed_open(orc_absorb(hy, (uint64_t)x));
                    out[((e * C + c) * H + y) * W + x] = (float)(low + (high[c] - low) * u);
                }
            }
        }
}
