// search_common.cuh -- query sources, box relations and the exact point predicates shared by
// the radius (K6) and kNN (K7) kernels.  FP64, compiled with -fmad=false: every expression is
// the reference's, evaluated left to right without contraction (geometry.hpp:127-231).
#pragma once

#include "lo_internal.cuh"

namespace lo {

enum Rel : int { kDisjoint = 0, kIntersects = 1, kContains = 2 };

// Queries: explicit SoA coordinates, optionally through a centre index array (cloud
// indices, as run_batch_loop's centres, search.cpp:287-312).
struct Queries {
    const double* x;
    const double* y;
    const double* z;
    const u32* idx;  // nullptr: query i is (x[i], y[i], z[i])
    u64 m;
};

__device__ __forceinline__ void load_query(const Queries& q, u64 i, double& cx, double& cy,
                                           double& cz) {
    const u64 j = q.idx ? q.idx[i] : i;
    cx = q.x[j];
    cy = q.y[j];
    cz = q.z[j];
}

struct NodeView {
    double lo[3], hi[3];
    u32 begin, end, child0, nchild;
};

__device__ __forceinline__ NodeView load_node(const TNode* __restrict__ tn, u32 t) {
    const double2* p = reinterpret_cast<const double2*>(tn + t);
    const double2 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2);
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(p + 3));
    NodeView v;
    v.lo[0] = a.x, v.lo[1] = a.y, v.lo[2] = b.x;
    v.hi[0] = b.y, v.hi[1] = c.x, v.hi[2] = c.y;
    v.begin = u.x, v.end = u.y, v.child0 = u.z, v.nchild = u.w;
    return v;
}

// geometry.hpp:162-169 axis_distances: near = max({lo - c, c - hi, 0}), far = max(c - lo, hi - c)
__device__ __forceinline__ double axis_near(double c, double lo, double hi) {
    const double a = lo - c, b = c - hi;
    double m = a < b ? b : a;
    return m < 0.0 ? 0.0 : m;
}
__device__ __forceinline__ double axis_far(double c, double lo, double hi) {
    const double a = c - lo, b = hi - c;
    return a < b ? b : a;
}

// kernel_octant_relation (geometry.hpp:197-231) on a box that contains the node's points.
template <int SHAPE>
__device__ __forceinline__ int relation(double cx, double cy, double cz, double r, double r2,
                                        const NodeView& nd) {
    const double nx = axis_near(cx, nd.lo[0], nd.hi[0]);
    const double ny = axis_near(cy, nd.lo[1], nd.hi[1]);
    const double fx = axis_far(cx, nd.lo[0], nd.hi[0]);
    const double fy = axis_far(cy, nd.lo[1], nd.hi[1]);
    double near_m, far_m, lim;
    if (SHAPE == LO_SPHERE || SHAPE == LO_CUBE) {
        const double nz = axis_near(cz, nd.lo[2], nd.hi[2]);
        const double fz = axis_far(cz, nd.lo[2], nd.hi[2]);
        if (SHAPE == LO_SPHERE) {
            near_m = nx * nx + ny * ny + nz * nz;
            far_m = fx * fx + fy * fy + fz * fz;
            lim = r2;
        } else {
            near_m = fmax(fmax(nx, ny), nz);
            far_m = fmax(fmax(fx, fy), fz);
            lim = r;
        }
    } else if (SHAPE == LO_CIRCLE) {
        near_m = nx * nx + ny * ny;
        far_m = fx * fx + fy * fy;
        lim = r2;
    } else {
        near_m = fmax(nx, ny);
        far_m = fmax(fx, fy);
        lim = r;
    }
    if (far_m < lim) return kContains;
    if (near_m >= lim) return kDisjoint;
    return kIntersects;
}

// kernel_contains (geometry.hpp:127-140): strict '<', dx = p - c.
template <int SHAPE>
__device__ __forceinline__ bool contains(double cx, double cy, double cz, double r, double r2,
                                         double px, double py, double pz) {
    const double dx = px - cx, dy = py - cy, dz = pz - cz;
    if (SHAPE == LO_SPHERE) return dx * dx + dy * dy + dz * dz < r2;
    if (SHAPE == LO_CIRCLE) return dx * dx + dy * dy < r2;
    if (SHAPE == LO_CUBE) return fmax(fmax(fabs(dx), fabs(dy)), fabs(dz)) < r;
    return fmax(fabs(dx), fabs(dy)) < r;
}

// octant_point_distance_sq (geometry.hpp:144-152) on a containing box: a lower bound of every
// member's point_dist_sq (search.cpp:180-185) under the same rounding.
__device__ __forceinline__ double box_dist_sq(double cx, double cy, double cz, const NodeView& nd) {
    const double gx = axis_near(cx, nd.lo[0], nd.hi[0]);
    const double gy = axis_near(cy, nd.lo[1], nd.hi[1]);
    const double gz = axis_near(cz, nd.lo[2], nd.hi[2]);
    return gx * gx + gy * gy + gz * gz;
}

// point_dist_sq (search.cpp:180-185): a = cloud point, b = centre.
__device__ __forceinline__ double point_dist_sq(double px, double py, double pz, double cx,
                                                double cy, double cz) {
    const double dx = px - cx, dy = py - cy, dz = pz - cz;
    return dx * dx + dy * dy + dz * dz;
}

constexpr int kStackCap = 192;  // DFS stack per warp: <= 7 * depth + 8 entries at depth <= 21

}  // namespace lo
