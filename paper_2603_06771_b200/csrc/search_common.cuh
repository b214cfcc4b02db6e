// search_common.cuh -- query sources, box relations and the exact point predicates shared by
// the radius (K6) and kNN (K7) kernels.  FP64, compiled with -fmad=false: every expression is
// the reference's, evaluated left to right without contraction (geometry.hpp:127-231).
#pragma once

#include <cmath>

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
    const float4* f = nullptr;  // FP32 copies (same indexing), for the filtered kernels
    double bmax = 0.0;          // >= |query - origin| on every axis
};

__device__ __forceinline__ float4 load_query_f(const Queries& q, u64 i) {
    const u64 j = q.idx ? q.idx[i] : i;
    return q.f[j];
}

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

// ---- FP32 filter with an exact FP64 band ------------------------------------------------
// Points and queries are also held as fl32(fl64(p - o)) (o = disc box min), node boxes as
// outward-rounded FP32 boxes.  With B >= |p - o| on every axis the per-axis error of any
// FP32 difference used below is <= d = 2 * 2^-23 * B + 2^-23 * 2r for values up to 2r, and a
// squared distance up to 4r^2 is off by at most
//     M = 1.25 * (3 * 2^-23 * 4r^2 + 2 sqrt(3) * 2r * d + 3 d^2 + 2^-49 * 4r^2)
// from the reference's FP64 value ((dx*dx + dy*dy) + dz*dz).  So d2_f < r^2 - M is a member,
// d2_f >= r^2 + M is not, and only the band in between is decided by the exact FP64
// predicate; values above 4r^2 are outside by the same argument (d < 0.01 r is required,
// else the filter is disabled and every test is exact).  Node boxes use the same margins
// for Contains (far_f < r^2 - M) and Disjoint (near_f >= r^2 + M).  DESIGN.md §4 has the
// derivation.
struct FloatTest {
    float t_lo, t_hi;  // squared-distance thresholds (Sphere, Circle)
    float r_lo, r_hi;  // L-inf thresholds (Cube, Square)
    int enabled;
    u32 coarse = 0;  // radius walk: internal nodes with at most this many points are taken whole
};

inline FloatTest make_float_test(double r, double bmax) {
    FloatTest f{};
    const double u = std::ldexp(1.0, -23);
    const double d = 2.0 * u * bmax + u * 2.0 * r;
    const double r2 = r * r;
    const double M = 1.25 * (3.0 * u * 4.0 * r2 + 2.0 * std::sqrt(3.0) * 2.0 * r * d + 3.0 * d * d +
                             std::ldexp(4.0 * r2, -49));
    const double ml = 1.25 * (d + std::ldexp(r, -50));
    f.enabled = (d < 0.01 * r) && (M < 0.25 * r2) && std::isfinite(M) && r2 < 1e30;
    if (!f.enabled) return f;
    auto down = [](double v) {
        float x = static_cast<float>(v);
        if (static_cast<double>(x) > v) x = std::nextafter(x, -INFINITY);
        return x;
    };
    auto up = [](double v) {
        float x = static_cast<float>(v);
        if (static_cast<double>(x) < v) x = std::nextafter(x, INFINITY);
        return x;
    };
    f.t_lo = down(r2 - M);
    f.t_hi = up(r2 + M);
    f.r_lo = down(r - ml);
    f.r_hi = up(r + ml);
    return f;
}

struct NodeF {
    float lo[3], hi[3];
    u32 begin, end, child0, nchild;
};

__device__ __forceinline__ NodeF load_node_f(const TNodeF* __restrict__ tf, u32 t) {
    const float4* p = reinterpret_cast<const float4*>(tf + t);
    const float4 a = __ldg(p), b = __ldg(p + 1);
    const uint4 c = __ldg(reinterpret_cast<const uint4*>(p + 2));
    NodeF v;
    v.lo[0] = a.x, v.lo[1] = a.y, v.lo[2] = a.z;
    v.hi[0] = b.x, v.hi[1] = b.y, v.hi[2] = b.z;
    v.begin = __float_as_uint(a.w), v.end = __float_as_uint(b.w);
    v.child0 = c.x, v.nchild = c.y;
    return v;
}

template <int SHAPE>
__device__ __forceinline__ int relation_f(const float4& q, const NodeF& nd, const FloatTest& ft) {
    const float nx = fmaxf(fmaxf(nd.lo[0] - q.x, q.x - nd.hi[0]), 0.f);
    const float ny = fmaxf(fmaxf(nd.lo[1] - q.y, q.y - nd.hi[1]), 0.f);
    const float fx = fmaxf(q.x - nd.lo[0], nd.hi[0] - q.x);
    const float fy = fmaxf(q.y - nd.lo[1], nd.hi[1] - q.y);
    if (SHAPE == LO_SPHERE || SHAPE == LO_CUBE) {
        const float nz = fmaxf(fmaxf(nd.lo[2] - q.z, q.z - nd.hi[2]), 0.f);
        const float fz = fmaxf(q.z - nd.lo[2], nd.hi[2] - q.z);
        if (SHAPE == LO_SPHERE) {
            if (fmaf(fz, fz, fmaf(fy, fy, fx * fx)) < ft.t_lo) return kContains;
            if (fmaf(nz, nz, fmaf(ny, ny, nx * nx)) >= ft.t_hi) return kDisjoint;
        } else {
            if (fmaxf(fmaxf(fx, fy), fz) < ft.r_lo) return kContains;
            if (fmaxf(fmaxf(nx, ny), nz) >= ft.r_hi) return kDisjoint;
        }
    } else if (SHAPE == LO_CIRCLE) {
        if (fmaf(fy, fy, fx * fx) < ft.t_lo) return kContains;
        if (fmaf(ny, ny, nx * nx) >= ft.t_hi) return kDisjoint;
    } else {
        if (fmaxf(fx, fy) < ft.r_lo) return kContains;
        if (fmaxf(nx, ny) >= ft.r_hi) return kDisjoint;
    }
    return kIntersects;
}

// Box-to-box test of a node against the tile's query box [bl, bh]: per axis the FP32 gap
// max(lo - bh, bl - hi, 0) is <= every tile query's own gap (FP32 subtraction is monotone),
// so "disjoint" here implies relation_f() == kDisjoint for every lane.
template <int SHAPE>
__device__ __forceinline__ bool tile_disjoint_f(const float* bl, const float* bh, const NodeF& nd,
                                                const FloatTest& ft) {
    const float gx = fmaxf(fmaxf(nd.lo[0] - bh[0], bl[0] - nd.hi[0]), 0.f);
    const float gy = fmaxf(fmaxf(nd.lo[1] - bh[1], bl[1] - nd.hi[1]), 0.f);
    if (SHAPE == LO_SPHERE || SHAPE == LO_CUBE) {
        const float gz = fmaxf(fmaxf(nd.lo[2] - bh[2], bl[2] - nd.hi[2]), 0.f);
        if (SHAPE == LO_SPHERE) return fmaf(gz, gz, fmaf(gy, gy, gx * gx)) >= ft.t_hi;
        return fmaxf(fmaxf(gx, gy), gz) >= ft.r_hi;
    }
    if (SHAPE == LO_CIRCLE) return fmaf(gy, gy, gx * gx) >= ft.t_hi;
    return fmaxf(gx, gy) >= ft.r_hi;
}

// relation_f()'s Disjoint half alone (one query against one node box).
template <int SHAPE>
__device__ __forceinline__ bool disjoint_f(const float4& q, const NodeF& nd, const FloatTest& ft) {
    const float nx = fmaxf(fmaxf(nd.lo[0] - q.x, q.x - nd.hi[0]), 0.f);
    const float ny = fmaxf(fmaxf(nd.lo[1] - q.y, q.y - nd.hi[1]), 0.f);
    if (SHAPE == LO_SPHERE || SHAPE == LO_CUBE) {
        const float nz = fmaxf(fmaxf(nd.lo[2] - q.z, q.z - nd.hi[2]), 0.f);
        if (SHAPE == LO_SPHERE) return fmaf(nz, nz, fmaf(ny, ny, nx * nx)) >= ft.t_hi;
        return fmaxf(fmaxf(nx, ny), nz) >= ft.r_hi;
    }
    if (SHAPE == LO_CIRCLE) return fmaf(ny, ny, nx * nx) >= ft.t_hi;
    return fmaxf(nx, ny) >= ft.r_hi;
}

// FP32 metric compared against the FloatTest thresholds: squared distance (Sphere, Circle)
// or L-inf distance (Cube, Square).
template <int SHAPE>
__device__ __forceinline__ float metric_f(const float4& q, const float4& p) {
    const float dx = p.x - q.x, dy = p.y - q.y;
    if (SHAPE == LO_SPHERE) {
        const float dz = p.z - q.z;
        return fmaf(dz, dz, fmaf(dy, dy, dx * dx));
    }
    if (SHAPE == LO_CIRCLE) return fmaf(dy, dy, dx * dx);
    if (SHAPE == LO_CUBE) return fmaxf(fmaxf(fabsf(dx), fabsf(dy)), fabsf(p.z - q.z));
    return fmaxf(fabsf(dx), fabsf(dy));
}

// 1 = member, 0 = not a member, 2 = inside the uncertainty band (decide in FP64)
template <int SHAPE>
__device__ __forceinline__ int classify_f(const float4& q, const float4& p, const FloatTest& ft) {
    const float dx = p.x - q.x, dy = p.y - q.y;
    if (SHAPE == LO_SPHERE || SHAPE == LO_CIRCLE) {
        float d2 = fmaf(dy, dy, dx * dx);
        if (SHAPE == LO_SPHERE) {
            const float dz = p.z - q.z;
            d2 = fmaf(dz, dz, d2);
        }
        return d2 < ft.t_lo ? 1 : (d2 >= ft.t_hi ? 0 : 2);
    } else {
        float m = fmaxf(fabsf(dx), fabsf(dy));
        if (SHAPE == LO_CUBE) m = fmaxf(m, fabsf(p.z - q.z));
        return m < ft.r_lo ? 1 : (m >= ft.r_hi ? 0 : 2);
    }
}

}  // namespace lo
