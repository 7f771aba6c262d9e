// Host-side BVH construction and packing for the B200 renderer.
//
// Replaces the reference's per-mesh build (bvh.py:68-136, a median split with
// leaf <= 4 and f64 flat arrays) with an SAH build (32 bins, exact sweep below 1024 triangles) whose output is packed
// for the GPU: every inner node is one 64-byte record holding BOTH children's
// fp32 boxes (so one record fetch tests two boxes) and triangles are 48-byte
// {v0, e1, e2} records. Boxes are padded outward so fp32 slab tests stay
// conservative (a node is never falsely culled).
#pragma once

#include <cstdint>
#include <vector>

namespace mdrt {

// Device record layouts (also used by the CPU visit counter in tests).
struct alignas(16) PackedNode {
    float c0x0, c0x1, c0y0, c0y1;  // child 0 box x/y  (lo, hi)
    float c1x0, c1x1, c1y0, c1y1;  // child 1 box x/y
    float c0z0, c0z1, c1z0, c1z1;  // both children z
    int32_t ref0, ref1;            // >= 0: inner node index; < 0: ~((first_tri << 3) | (count-1))
    int32_t pad0, pad1;
};
static_assert(sizeof(PackedNode) == 64, "node record must be 64 B");

struct alignas(16) PackedTri {
    float v0x, v0y, v0z, id;       // id: original face index (bit pattern of int32)
    float e1x, e1y, e1z, pad1;
    float e2x, e2y, e2z, pad2;
};
static_assert(sizeof(PackedTri) == 48, "triangle record must be 48 B");

constexpr int kMaxLeafTris = 4;   // default leaf size bound (encoding allows 8)
constexpr int kMaxDepth = 24;   // builder guarantees leaf depth <= kMaxDepth (= GPU stack size)

inline int32_t leaf_ref(int64_t first, int count) {
    return ~static_cast<int32_t>((first << 3) | (count - 1));
}

struct PackedTree {
    std::vector<PackedNode> nodes;   // node 0 is the root
    std::vector<PackedTri> tris;
    std::vector<int64_t> tri_index;  // packed triangle -> original face index
    int depth = 0;                   // max leaf depth (root = 0)
    double center[3] = {0, 0, 0};    // bounding sphere (local frame)
    double radius = 0;
    double box_lo[3] = {0, 0, 0};    // exact AABB of the referenced vertices (local frame)
    double box_hi[3] = {0, 0, 0};
};

// Build + pack one mesh. verts (nv,3) f64, faces (nf,3) i64. Faces must be
// valid indices. Node refs/triangle refs are relative to this tree; the caller
// offsets them when concatenating trees (offset_tree).
// leaf_max <= 0: the default leaf bound (kMaxLeafTris, or MDRT_LEAF_MAX).
PackedTree build_tree(const double* verts, int64_t nv, const int64_t* faces, int64_t nf, int leaf_max = 0);

// Shift a tree's internal node and triangle references by the given offsets.
void offset_tree(PackedTree& t, int32_t node_off, int32_t tri_off);

}  // namespace mdrt
