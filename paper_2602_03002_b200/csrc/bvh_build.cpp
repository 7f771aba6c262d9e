// SAH BVH build (32-bin SAH; exact sweep SAH for small nodes) + GPU packing (see bvh_build.h).
#include "bvh_build.h"

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

namespace mdrt {
namespace {

struct Box {
    double lo[3] = {std::numeric_limits<double>::infinity(), std::numeric_limits<double>::infinity(),
                    std::numeric_limits<double>::infinity()};
    double hi[3] = {-std::numeric_limits<double>::infinity(), -std::numeric_limits<double>::infinity(),
                    -std::numeric_limits<double>::infinity()};
    void grow(const Box& b) {
        for (int a = 0; a < 3; ++a) {
            lo[a] = std::min(lo[a], b.lo[a]);
            hi[a] = std::max(hi[a], b.hi[a]);
        }
    }
    void grow(const double* p) {
        for (int a = 0; a < 3; ++a) {
            lo[a] = std::min(lo[a], p[a]);
            hi[a] = std::max(hi[a], p[a]);
        }
    }
    bool empty() const { return lo[0] > hi[0]; }
    double area() const {
        if (empty()) return 0.0;
        double dx = hi[0] - lo[0], dy = hi[1] - lo[1], dz = hi[2] - lo[2];
        return 2.0 * (dx * dy + dy * dz + dz * dx);
    }
};

struct BNode {
    Box box;
    int32_t child[2] = {-1, -1};  // build-node indices, -1 for leaves
    int64_t first = 0, count = 0;
    int depth = 0;
    bool sorted = false;   // ord3_[a][first, first + count) hold this node's triangles by centroid a
};

constexpr int kBins = 32;
constexpr double kCostTri = 1.0;   // relative cost of one triangle test

// SAH node cost relative to a triangle test (one 64 B record = two box tests)
// and the largest leaf; overridable for tuning experiments via
// MDRT_SAH_NODE_COST / MDRT_LEAF_MAX (<= 8, the leaf encoding's limit).
struct BuildOptions {
    double node_cost = 1.2;            // < 0 / 0 below: chosen per mesh size (large_mesh_*)
    int leaf_max = kMaxLeafTris;
    bool node_cost_set = false, leaf_max_set = false;
    // nodes with <= sweep_max triangles take the exact sweep SAH (every split of the
    // centroid order on every axis) instead of 32 bins: config 3 (8,750-triangle
    // stepping-stone terrain, large box faces) +6.0 %, configs 2 and paper +-0.1 %;
    // 4096 / 16384 / all nodes gained no more and cost build time (config 5: 7 -> 17 s
    // at 16384)
    int64_t sweep_max = 1024;
};

const BuildOptions& options() {
    static const BuildOptions o = [] {
        BuildOptions r;
        if (const char* v = std::getenv("MDRT_SAH_NODE_COST")) {
            r.node_cost = std::atof(v);
            r.node_cost_set = true;
        }
        if (const char* v = std::getenv("MDRT_LEAF_MAX")) {
            r.leaf_max = std::min(8, std::max(1, std::atoi(v)));
            r.leaf_max_set = true;
        }
        if (const char* v = std::getenv("MDRT_SAH_SWEEP")) r.sweep_max = std::atoll(v);
        return r;
    }();
    return o;
}

// Large meshes (>= 500k triangles) get a costlier node and leaves of up to 8
// triangles: their trees are deep, and a node visit loads the L1 data pipe while
// triangle tests run on the otherwise idle texture pipe. Measured (round 2,
// profiles/experiments/r02_sah_large_mesh.txt): config 5 (3.37M triangles) +2.6 %,
// its 1M-triangle variant +2.8 %; the same setting on config 2 (259k) -0.2 %,
// config 3 (8.75k) -3.0 %, paper (259k) -1.4 %, hence the size bound.
constexpr int64_t kLargeMesh = 500000;
double node_cost_for(int64_t nf) {
    const BuildOptions& o = options();
    return o.node_cost_set ? o.node_cost : (nf >= kLargeMesh ? 2.0 : o.node_cost);
}
int default_leaf_max(int64_t nf) {
    const BuildOptions& o = options();
    return o.leaf_max_set ? o.leaf_max : (nf >= kLargeMesh ? 8 : o.leaf_max);
}

class Builder {
   public:
    Builder(const std::vector<Box>& tb, const std::vector<std::array<double, 3>>& cen, int leaf_max)
        : tbox_(tb), cen_(cen), leaf_max_(leaf_max),
          node_cost_(node_cost_for(static_cast<int64_t>(tb.size()))) {}

    std::vector<BNode> nodes;
    std::vector<int64_t> idx;

    void run() {
        const int64_t F = static_cast<int64_t>(tbox_.size());
        idx.resize(F);
        for (int64_t i = 0; i < F; ++i) idx[i] = i;
        nodes.reserve(2 * F);
        BNode root;
        root.first = 0;
        root.count = F;
        root.depth = 0;
        for (int64_t i = 0; i < F; ++i) root.box.grow(tbox_[i]);
        nodes.push_back(root);
        std::vector<int32_t> stack{0};
        while (!stack.empty()) {
            int32_t ni = stack.back();
            stack.pop_back();
            int32_t kids[2];
            if (split(ni, kids)) {
                stack.push_back(kids[1]);
                stack.push_back(kids[0]);
            }
        }
    }

   private:
    const std::vector<Box>& tbox_;
    const std::vector<std::array<double, 3>>& cen_;
    const int leaf_max_;
    const double node_cost_;
    // sweep SAH state: per axis, the triangles of every node in the sweep region
    // in centroid order (ties by index), kept through splits by stable partition
    std::vector<int64_t> ord3_[3];
    std::vector<uint8_t> left_;          // per triangle: in the left child of the current split
    std::vector<int64_t> scratch_;
    std::vector<double> sweep_area_;
    std::vector<std::pair<double, int64_t>> sweep_key_;

    // ord3_[a][first, first + n) = idx[first, first + n) ordered by centroid a
    void sort_segment(int a, int64_t first, int64_t n) {
        sweep_key_.resize(n);
        for (int64_t i = 0; i < n; ++i) sweep_key_[i] = {cen_[idx[first + i]][a], idx[first + i]};
        std::sort(sweep_key_.begin(), sweep_key_.end());
        for (int64_t i = 0; i < n; ++i) ord3_[a][first + i] = sweep_key_[i].second;
    }

    // Returns true and fills kids when node ni was split.
    bool split(int32_t ni, int32_t kids[2]) {
        const int64_t first = nodes[ni].first, n = nodes[ni].count;
        const int depth = nodes[ni].depth;
        if (n <= 1) return false;
        Box cb;  // centroid bounds
        for (int64_t i = first; i < first + n; ++i) cb.grow(cen_[idx[i]].data());
        int64_t mid = -1;
        bool kids_sorted = false;   // the sweep split kept ord3_ valid for both children
        // Switch to object-median splits when the remaining depth budget gets
        // tight: a median tree below this node adds ceil(log2(n)) levels.
        int need = 0;
        const int leaf_max = leaf_max_;
        while ((int64_t(leaf_max) << need) < n) ++need;
        const bool force_median = depth + need + 1 >= kMaxDepth;
        if (!force_median && n <= options().sweep_max) {
            // exact SAH: every split position of the centroid order on every axis
            double best_cost = std::numeric_limits<double>::infinity();
            int best_axis = -1;
            int64_t best_pos = -1;
            const double parent_area = nodes[ni].box.area();
            std::vector<double>& right_area = sweep_area_;
            right_area.resize(n);
            if (!nodes[ni].sorted) {
                for (int a = 0; a < 3; ++a) {
                    if (ord3_[a].empty()) ord3_[a].resize(idx.size());
                    sort_segment(a, first, n);
                }
            }
            for (int a = 0; a < 3; ++a) {
                if (!(cb.hi[a] - cb.lo[a] > 0.0)) continue;
                const int64_t* ord = ord3_[a].data() + first;
                Box acc;
                for (int64_t i = n - 1; i > 0; --i) {
                    acc.grow(tbox_[ord[i]]);
                    right_area[i] = acc.area();
                }
                Box lacc;
                for (int64_t i = 1; i < n; ++i) {
                    lacc.grow(tbox_[ord[i - 1]]);
                    const double cost = node_cost_ +
                                        (lacc.area() * i + right_area[i] * (n - i)) * kCostTri /
                                            std::max(parent_area, 1e-300);
                    if (cost < best_cost) {
                        best_cost = cost;
                        best_axis = a;
                        best_pos = i;
                    }
                }
            }
            const double leaf_cost = kCostTri * static_cast<double>(n);
            if (n <= leaf_max && !(best_cost < leaf_cost)) return false;
            if (best_axis >= 0) {
                const int k = best_axis;
                std::copy(ord3_[k].begin() + first, ord3_[k].begin() + first + n, idx.begin() + first);
                mid = first + best_pos;
                // the other axes' orders: stable partition into left then right
                if (left_.empty()) left_.resize(idx.size());
                for (int64_t i = first; i < first + n; ++i) left_[idx[i]] = i < mid ? 1 : 0;
                scratch_.resize(n);
                for (int a = 0; a < 3; ++a) {
                    if (a == k) continue;
                    int64_t* o = ord3_[a].data() + first;
                    int64_t l = 0, r = best_pos;
                    for (int64_t i = 0; i < n; ++i) scratch_[left_[o[i]] ? l++ : r++] = o[i];
                    std::copy(scratch_.begin(), scratch_.end(), o);
                }
                kids_sorted = true;
            }
        } else if (!force_median) {
            double best_cost = std::numeric_limits<double>::infinity();
            int best_axis = -1, best_bin = -1;
            const double parent_area = nodes[ni].box.area();
            for (int a = 0; a < 3; ++a) {
                const double ext = cb.hi[a] - cb.lo[a];
                if (!(ext > 0.0)) continue;
                Box bb[kBins];
                int64_t bc[kBins] = {0};
                const double scale = kBins / ext;
                for (int64_t i = first; i < first + n; ++i) {
                    int b = static_cast<int>((cen_[idx[i]][a] - cb.lo[a]) * scale);
                    b = std::min(std::max(b, 0), kBins - 1);
                    bb[b].grow(tbox_[idx[i]]);
                    ++bc[b];
                }
                double right_area[kBins];
                int64_t right_cnt[kBins];
                Box acc;
                int64_t cnt = 0;
                for (int b = kBins - 1; b > 0; --b) {
                    acc.grow(bb[b]);
                    cnt += bc[b];
                    right_area[b] = acc.area();
                    right_cnt[b] = cnt;
                }
                Box lacc;
                int64_t lcnt = 0;
                for (int b = 0; b < kBins - 1; ++b) {
                    lacc.grow(bb[b]);
                    lcnt += bc[b];
                    if (lcnt == 0 || right_cnt[b + 1] == 0) continue;
                    double cost = node_cost_ + (lacc.area() * lcnt + right_area[b + 1] * right_cnt[b + 1]) *
                                                  kCostTri / std::max(parent_area, 1e-300);
                    if (cost < best_cost) {
                        best_cost = cost;
                        best_axis = a;
                        best_bin = b;
                    }
                }
            }
            const double leaf_cost = kCostTri * static_cast<double>(n);
            if (n <= leaf_max && !(best_cost < leaf_cost)) return false;
            if (best_axis >= 0) {
                const double ext = cb.hi[best_axis] - cb.lo[best_axis];
                const double scale = kBins / ext;
                auto* beg = idx.data() + first;
                auto* end = beg + n;
                auto* m = std::partition(beg, end, [&](int64_t t) {
                    int b = static_cast<int>((cen_[t][best_axis] - cb.lo[best_axis]) * scale);
                    b = std::min(std::max(b, 0), kBins - 1);
                    return b <= best_bin;
                });
                mid = first + (m - beg);
                if (mid == first || mid == first + n) mid = -1;
            }
        }
        if (mid < 0) {
            if (n <= leaf_max && !force_median) return false;
            // object median on the longest centroid axis (or index median)
            int axis = 0;
            double ext = cb.hi[0] - cb.lo[0];
            for (int a = 1; a < 3; ++a)
                if (cb.hi[a] - cb.lo[a] > ext) { ext = cb.hi[a] - cb.lo[a]; axis = a; }
            mid = first + n / 2;
            if (ext > 0.0) {
                std::nth_element(idx.begin() + first, idx.begin() + mid, idx.begin() + first + n,
                                 [&](int64_t x, int64_t y) {
                                     if (cen_[x][axis] != cen_[y][axis]) return cen_[x][axis] < cen_[y][axis];
                                     return x < y;
                                 });
            }
            if (n <= leaf_max && force_median) {
                // tiny node deep in the tree: a leaf is fine
                return false;
            }
        }
        for (int k = 0; k < 2; ++k) {
            BNode c;
            c.first = k == 0 ? first : mid;
            c.count = k == 0 ? mid - first : first + n - mid;
            c.depth = depth + 1;
            c.sorted = kids_sorted;
            for (int64_t i = c.first; i < c.first + c.count; ++i) c.box.grow(tbox_[idx[i]]);
            kids[k] = static_cast<int32_t>(nodes.size());
            nodes.push_back(c);
        }
        nodes[ni].child[0] = kids[0];
        nodes[ni].child[1] = kids[1];
        return true;
    }
};

// Round a box outward to fp32 with a conservative pad (see bvh_build.h).
void pad_box(const Box& b, float lo[3], float hi[3]) {
    for (int a = 0; a < 3; ++a) {
        if (b.empty()) {
            lo[a] = std::numeric_limits<float>::infinity();
            hi[a] = -std::numeric_limits<float>::infinity();
            continue;
        }
        const double mag = std::max(std::fabs(b.lo[a]), std::fabs(b.hi[a]));
        const double pad = 2e-5 + mag * (1.0 / (1 << 20));
        lo[a] = std::nextafter(static_cast<float>(b.lo[a] - pad), -std::numeric_limits<float>::infinity());
        hi[a] = std::nextafter(static_cast<float>(b.hi[a] + pad), std::numeric_limits<float>::infinity());
    }
}

}  // namespace

PackedTree build_tree(const double* verts, int64_t nv, const int64_t* faces, int64_t nf, int leaf_max) {
    if (leaf_max <= 0) leaf_max = default_leaf_max(nf);
    if (leaf_max > 8) throw std::invalid_argument("leaf size must be <= 8 (leaf encoding)");
    if (nf <= 0) throw std::invalid_argument("cannot build a BVH over an empty mesh");
    // The traversal stack holds kMaxDepth entries. The builder keeps every leaf
    // within kMaxDepth levels by switching to median splits when the remaining
    // depth budget gets tight, which is only possible while the mesh fits a
    // complete tree of leaf_max-triangle leaves: reject larger meshes here
    // instead of overflowing the device stack (bvh.py:68-136 has no depth bound:
    // its CPU stack is 128 entries, numba_backend.py:126).
    if (nf > (static_cast<int64_t>(leaf_max) << (kMaxDepth - 1)))
        throw std::invalid_argument("mesh too large for the traversal stack (more than leaf_max * 2^" +
                                    std::to_string(kMaxDepth - 1) + " triangles): split it into several bodies");
    for (int64_t i = 0; i < 3 * nv; ++i)
        if (!std::isfinite(verts[i])) throw std::invalid_argument("mesh vertices must be finite");
    std::vector<Box> tb(nf);
    std::vector<std::array<double, 3>> cen(nf);
    for (int64_t f = 0; f < nf; ++f) {
        for (int k = 0; k < 3; ++k) {
            int64_t vi = faces[f * 3 + k];
            if (vi < 0 || vi >= nv) throw std::invalid_argument("face index out of range");
            tb[f].grow(verts + vi * 3);
        }
        for (int a = 0; a < 3; ++a) cen[f][a] = 0.5 * (tb[f].lo[a] + tb[f].hi[a]);
    }
    Builder bld(tb, cen, leaf_max);
    bld.run();

    PackedTree out;
    // triangles in leaf order (DFS), assigned during packing
    out.tris.reserve(nf);
    out.tri_index.reserve(nf);

    // Pack inner nodes in DFS order; leaves are referenced from their parent.
    std::vector<int32_t> packed_of(bld.nodes.size(), -1);
    auto emit_leaf = [&](const BNode& n) -> int32_t {
        const int64_t first = static_cast<int64_t>(out.tris.size());
        for (int64_t i = n.first; i < n.first + n.count; ++i) {
            const int64_t f = bld.idx[i];
            const double* a = verts + faces[f * 3 + 0] * 3;
            const double* b = verts + faces[f * 3 + 1] * 3;
            const double* c = verts + faces[f * 3 + 2] * 3;
            PackedTri t{};
            t.v0x = static_cast<float>(a[0]);
            t.v0y = static_cast<float>(a[1]);
            t.v0z = static_cast<float>(a[2]);
            int32_t id32 = static_cast<int32_t>(f);
            std::memcpy(&t.id, &id32, 4);
            t.e1x = static_cast<float>(b[0] - a[0]);
            t.e1y = static_cast<float>(b[1] - a[1]);
            t.e1z = static_cast<float>(b[2] - a[2]);
            t.e2x = static_cast<float>(c[0] - a[0]);
            t.e2y = static_cast<float>(c[1] - a[1]);
            t.e2z = static_cast<float>(c[2] - a[2]);
            out.tris.push_back(t);
            out.tri_index.push_back(f);
        }
        if (n.count > 8) throw std::logic_error("leaf too large");
        return leaf_ref(first, static_cast<int>(n.count));
    };

    int maxdepth = 0;
    const BNode& root = bld.nodes[0];
    if (root.child[0] < 0) {
        // whole mesh is one leaf: root record with an empty second child
        PackedNode pn{};
        float lo[3], hi[3];
        pad_box(root.box, lo, hi);
        pn.c0x0 = lo[0]; pn.c0x1 = hi[0]; pn.c0y0 = lo[1]; pn.c0y1 = hi[1]; pn.c0z0 = lo[2]; pn.c0z1 = hi[2];
        Box empty;
        pad_box(empty, lo, hi);
        pn.c1x0 = lo[0]; pn.c1x1 = hi[0]; pn.c1y0 = lo[1]; pn.c1y1 = hi[1]; pn.c1z0 = lo[2]; pn.c1z1 = hi[2];
        out.nodes.push_back(pn);
        out.nodes[0].ref0 = emit_leaf(root);
        out.nodes[0].ref1 = leaf_ref(0, 1);  // never reached: empty box
        maxdepth = 1;
    } else {
        // iterative DFS: allocate record, then fill children refs
        struct Item { int32_t b; int32_t packed; };
        std::vector<Item> st;
        out.nodes.push_back(PackedNode{});
        st.push_back({0, 0});
        while (!st.empty()) {
            Item it = st.back();
            st.pop_back();
            const BNode& n = bld.nodes[it.b];
            maxdepth = std::max(maxdepth, n.depth + 1);
            PackedNode pn{};
            float lo[3], hi[3];
            const BNode& a = bld.nodes[n.child[0]];
            const BNode& b = bld.nodes[n.child[1]];
            pad_box(a.box, lo, hi);
            pn.c0x0 = lo[0]; pn.c0x1 = hi[0]; pn.c0y0 = lo[1]; pn.c0y1 = hi[1]; pn.c0z0 = lo[2]; pn.c0z1 = hi[2];
            pad_box(b.box, lo, hi);
            pn.c1x0 = lo[0]; pn.c1x1 = hi[0]; pn.c1y0 = lo[1]; pn.c1y1 = hi[1]; pn.c1z0 = lo[2]; pn.c1z1 = hi[2];
            int32_t refs[2];
            int32_t pending[2] = {-1, -1};
            for (int k = 0; k < 2; ++k) {
                const BNode& c = bld.nodes[n.child[k]];
                if (c.child[0] < 0) {
                    refs[k] = emit_leaf(c);
                } else {
                    refs[k] = static_cast<int32_t>(out.nodes.size());
                    out.nodes.push_back(PackedNode{});
                    pending[k] = refs[k];
                }
            }
            pn.ref0 = refs[0];
            pn.ref1 = refs[1];
            out.nodes[it.packed] = pn;
            // child 0 visited first (pushed last)
            if (pending[1] >= 0) st.push_back({n.child[1], pending[1]});
            if (pending[0] >= 0) st.push_back({n.child[0], pending[0]});
        }
    }
    out.depth = maxdepth;
    if (out.depth > kMaxDepth)   // cannot happen given the size check above; never ship a deeper tree
        throw std::invalid_argument("BVH deeper than the traversal stack");

    // bounding sphere of the vertices actually referenced
    Box all = root.box;
    for (int a = 0; a < 3; ++a) {
        out.center[a] = 0.5 * (all.lo[a] + all.hi[a]);
        out.box_lo[a] = all.lo[a];
        out.box_hi[a] = all.hi[a];
    }
    double r2 = 0.0;
    for (int64_t f = 0; f < nf; ++f)
        for (int k = 0; k < 3; ++k) {
            const double* p = verts + faces[f * 3 + k] * 3;
            double dx = p[0] - out.center[0], dy = p[1] - out.center[1], dz = p[2] - out.center[2];
            r2 = std::max(r2, dx * dx + dy * dy + dz * dz);
        }
    out.radius = std::sqrt(r2) * (1.0 + 1e-6) + 1e-4;
    return out;
}

void offset_tree(PackedTree& t, int32_t node_off, int32_t tri_off) {
    for (auto& n : t.nodes) {
        int32_t* refs[2] = {&n.ref0, &n.ref1};
        for (int32_t* r : refs) {
            if (*r >= 0) {
                *r += node_off;
            } else {
                int32_t v = ~*r;
                int64_t first = (v >> 3) + tri_off;
                int count = (v & 7) + 1;
                *r = leaf_ref(first, count);
            }
        }
    }
}

}  // namespace mdrt
