// radius_struct.cu -- RadiusMethod::Struct: neighbours_struct (search.cpp:76-135) batched.
//
// The reference's Struct result is defined by ITS octant boxes: a node whose padded octant box
// (octant_bounds, sfc.cpp:110-127) lies strictly inside the kernel contributes its whole
// [begin, end) as a range (adjacent ranges coalesce, search.cpp:124-129), a Disjoint box
// prunes, and the points of the remaining leaves are tested one by one ("singles").  So unlike
// Lin/Prune -- where any box containing the points gives the same index set -- the ranges /
// singles split must be computed on exactly those boxes: tnode_ref_boxes (octree.cu)
// materialises them once per tree.
//
// One warp owns 32 consecutive queries and walks the union of their traversals (children in
// code order == the reference's pop order, search.cpp:30-41); each lane classifies every
// visited node for its own query with the FP64 kernel_octant_relation, and a lane whose query
// contains a node ignores that node's descendants (their begin lies inside the emitted range).
// Count pass -> three u64 scans (members, ranges, singles) -> fill pass -> row digests
// hashed like search.cpp:325-336.
#include <algorithm>

#include "radius_float.cuh"

namespace lo {

template <int SHAPE, bool FILL>
__global__ void __launch_bounds__(kRadiusThreads) radius_struct_kernel(
    const TNode* __restrict__ tn, const double* __restrict__ rb, const double* __restrict__ px,
    const double* __restrict__ py, const double* __restrict__ pz, Queries q, double r, double r2,
    u32* __restrict__ counts, u32* __restrict__ nrng, u32* __restrict__ nsgl,
    const u64* __restrict__ r_off, u32* __restrict__ ranges, const u64* __restrict__ s_off,
    u32* __restrict__ singles) {
    __shared__ u32 stack_s[kRadiusWarps][kStackCap];
    __shared__ double sx[kRadiusWarps][32], sy[kRadiusWarps][32], sz[kRadiusWarps][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    u32* stack = stack_s[w];
    const u64 ntiles = (q.m + 31) / 32;
    for (u64 tile = static_cast<u64>(blockIdx.x) * kRadiusWarps + w; tile < ntiles;
         tile += static_cast<u64>(gridDim.x) * kRadiusWarps) {
        const u64 qi = tile * 32 + lane;
        const bool active = qi < q.m;
        double cx = 0.0, cy = 0.0, cz = 0.0;
        if (active) load_query(q, qi, cx, cy, cz);
        u32 count = 0, nr = 0, ns = 0;
        u32 last_e = 0;     // end of the last emitted range (valid when nr > 0)
        u32 skip_end = 0;   // descendants of an emitted node start below this
        u32* rrow = nullptr;
        u32* srow = nullptr;
        if (FILL && active) {
            rrow = ranges + 2 * r_off[qi];
            srow = singles + s_off[qi];
        }
        int sp = 1;
        if (lane == 0) stack[0] = 0;
        __syncwarp();
        while (sp > 0) {
            const u32 t = stack[--sp];
            const uint4 u = __ldg(reinterpret_cast<const uint4*>(tn + t) + 3);
            const u32 nb = u.x, ne = u.y, child0 = u.z, nchild = u.w;
            int rel = kDisjoint;
            if (active && nb >= skip_end) {
                NodeView box;
                const double* b = rb + 6 * static_cast<u64>(t);
#pragma unroll
                for (int a = 0; a < 3; ++a) box.lo[a] = __ldg(b + a), box.hi[a] = __ldg(b + 3 + a);
                rel = relation<SHAPE>(cx, cy, cz, r, r2, box);
            }
            if (rel == kContains) {
                if (nr > 0 && last_e == nb) {  // adjacent contained octants coalesce
                    if (FILL) rrow[2 * (nr - 1) + 1] = ne;
                } else {
                    if (FILL) rrow[2 * nr] = nb, rrow[2 * nr + 1] = ne;
                    ++nr;
                }
                last_e = ne;
                count += ne - nb;
                skip_end = ne;
            }
            const unsigned hit = __ballot_sync(~0u, rel == kIntersects);
            if (!hit) continue;
            if (nchild == 0) {
                for (u32 base = nb; base < ne; base += 32) {
                    const u32 j = base + lane;
                    __syncwarp();
                    if (j < ne) {
                        sx[w][lane] = px[j];
                        sy[w][lane] = py[j];
                        sz[w][lane] = pz[j];
                    }
                    __syncwarp();
                    if (rel == kIntersects) {
                        const u32 cnt = min(32u, ne - base);
                        for (u32 jj = 0; jj < cnt; ++jj) {
                            if (contains<SHAPE>(cx, cy, cz, r, r2, sx[w][jj], sy[w][jj], sz[w][jj])) {
                                if (FILL) srow[ns] = base + jj;
                                ++ns;
                                ++count;
                            }
                        }
                    }
                }
            } else {
                __syncwarp();
                if (lane < static_cast<int>(nchild)) stack[sp + nchild - 1 - lane] = child0 + lane;
                sp += nchild;
                __syncwarp();
            }
        }
        if (!FILL && active) {
            counts[qi] = count;
            nrng[qi] = nr;
            nsgl[qi] = ns;
        }
        __syncwarp();
    }
}

// Struct row digest (search.cpp:325-336): ranges as begin << 32 | end, a separator, singles.
__global__ void struct_digest(const u64* __restrict__ r_off, const u32* __restrict__ ranges,
                              const u64* __restrict__ s_off, const u32* __restrict__ singles, u64 m,
                              u64* __restrict__ fps) {
    for (u64 row = blockIdx.x * (u64)blockDim.x + threadIdx.x; row < m;
         row += (u64)gridDim.x * blockDim.x) {
        u64 h = kFnvOffset;
        for (u64 j = r_off[row]; j < r_off[row + 1]; ++j)
            h = fnv_u64(h, (static_cast<u64>(ranges[2 * j]) << 32) | ranges[2 * j + 1]);
        h = fnv_u64(h, ~0ull);
        for (u64 j = s_off[row]; j < s_off[row + 1]; ++j) h = fnv_u32(h, singles[j]);
        fps[row] = h;
    }
}

// RangedResult::expand (search.hpp:45-49): merge ranges and singles into ascending indices.
__global__ void struct_expand(const u64* __restrict__ r_off, const u32* __restrict__ ranges,
                              const u64* __restrict__ s_off, const u32* __restrict__ singles,
                              const u64* __restrict__ offsets, u64 m, u32* __restrict__ out) {
    for (u64 row = blockIdx.x * (u64)blockDim.x + threadIdx.x; row < m;
         row += (u64)gridDim.x * blockDim.x) {
        u64 ri = r_off[row], re = r_off[row + 1], si = s_off[row], se = s_off[row + 1];
        u32* o = out + offsets[row];
        while (ri < re || si < se) {
            if (si == se || (ri < re && ranges[2 * ri] < singles[si])) {
                for (u32 i = ranges[2 * ri]; i < ranges[2 * ri + 1]; ++i) *o++ = i;
                ++ri;
            } else {
                *o++ = singles[si++];
            }
        }
    }
}

static int grid_rows(lo_context* ctx, u64 m) {
    return static_cast<int>(std::max<u64>(1, std::min<u64>((m + 255) / 256, ctx->sm_count * 16ull)));
}

template <bool FILL>
static void launch_struct(lo_context* ctx, int shape, const lo_octree* t, const lo_coded* c,
                          const Queries& q, double r, lo_csr* out, u32* nrng, u32* nsgl) {
    const double r2 = r * r;  // SearchKernel ctor (geometry.hpp:107)
    const u64 tiles = (q.m + 31) / 32;
    const int blocks = static_cast<int>(std::max<u64>(
        1, std::min<u64>((tiles + kRadiusWarps - 1) / kRadiusWarps, static_cast<u64>(ctx->sm_count) * 64)));
#define LO_STRUCT_CASE(S)                                                                         \
    case S:                                                                                       \
        radius_struct_kernel<S, FILL><<<blocks, kRadiusThreads, 0, ctx->stream>>>(                \
            t->tn, t->rb, c->x, c->y, c->z, q, r, r2, out->counts, nrng, nsgl, out->range_offsets, \
            out->ranges, out->single_offsets, out->singles);                                      \
        break;
    switch (shape) {
        LO_STRUCT_CASE(LO_SPHERE)
        LO_STRUCT_CASE(LO_CIRCLE)
        LO_STRUCT_CASE(LO_CUBE)
        LO_STRUCT_CASE(LO_SQUARE)
        default: throw Error(LO_INVALID_ARGUMENT, "unknown kernel shape");
    }
#undef LO_STRUCT_CASE
    LO_CHECK_LAUNCH();
}

lo_csr* radius_struct_search(lo_context* ctx, const lo_octree* t, const lo_coded* c, int shape,
                             double r, const Queries& q, bool fingerprint) {
    require(t != nullptr && c != nullptr, LO_INVALID_ARGUMENT, "null tree or cloud");
    require(r > 0.0 && std::isfinite(r), LO_INVALID_ARGUMENT,
            "kernel radius must be positive and finite");
    require(shape >= LO_SPHERE && shape <= LO_SQUARE, LO_INVALID_ARGUMENT, "unknown kernel shape");
    ensure_ref_boxes(ctx, c, t);
    auto* out = new lo_csr;
    out->ctx = ctx;
    out->rows = q.m;
    out->is_struct = true;
    u32 *nrng = nullptr, *nsgl = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    try {
        LO_CUDA(cudaEventCreate(&e0));
        LO_CUDA(cudaEventCreate(&e1));
        LO_CUDA(cudaEventRecord(e0, ctx->stream));
        out->counts = dalloc_t<u32>(ctx, q.m);
        out->offsets = dalloc_t<u64>(ctx, q.m + 1);
        out->range_offsets = dalloc_t<u64>(ctx, q.m + 1);
        out->single_offsets = dalloc_t<u64>(ctx, q.m + 1);
        nrng = dalloc_t<u32>(ctx, q.m);
        nsgl = dalloc_t<u32>(ctx, q.m);
        stage_begin(ctx, "struct_count");
        if (q.m) launch_struct<false>(ctx, shape, t, c, q, r, out, nrng, nsgl);
        stage_end(ctx);
        exclusive_scan_u32_to_u64(ctx, out->counts, out->offsets, q.m);
        exclusive_scan_u32_to_u64(ctx, nrng, out->range_offsets, q.m);
        exclusive_scan_u32_to_u64(ctx, nsgl, out->single_offsets, q.m);
        out->total = read_scalar(ctx, out->offsets + q.m);
        out->total_ranges = read_scalar(ctx, out->range_offsets + q.m);
        out->total_singles = read_scalar(ctx, out->single_offsets + q.m);
        out->ranges = dalloc_t<u32>(ctx, 2 * out->total_ranges);
        out->singles = dalloc_t<u32>(ctx, out->total_singles);
        stage_begin(ctx, "struct_fill");
        if (q.m) launch_struct<true>(ctx, shape, t, c, q, r, out, nrng, nsgl);
        stage_end(ctx);
        if (fingerprint) {
            out->fps = dalloc_t<u64>(ctx, q.m);
            if (q.m) {
                struct_digest<<<grid_rows(ctx, q.m), 256, 0, ctx->stream>>>(
                    out->range_offsets, out->ranges, out->single_offsets, out->singles, q.m, out->fps);
                LO_CHECK_LAUNCH();
            }
        }
        LO_CUDA(cudaEventRecord(e1, ctx->stream));
        sync(ctx);
        LO_CUDA(cudaEventElapsedTime(&out->ms, e0, e1));
        out->mean = q.m ? static_cast<double>(out->total) / static_cast<double>(q.m) : 0.0;
    } catch (...) {
        dfree(ctx, nrng);
        dfree(ctx, nsgl);
        free_csr_buffers(ctx, out);
        delete out;
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
        throw;
    }
    dfree(ctx, nrng);
    dfree(ctx, nsgl);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return out;
}

// The expanded CSR of a Struct result (RangedResult::expand per row), built on first use.
void ensure_expanded(lo_context* ctx, lo_csr* csr) {
    if (!csr->is_struct || csr->indices || csr->total == 0) return;
    csr->indices = dalloc_t<u32>(ctx, csr->total);
    struct_expand<<<grid_rows(ctx, csr->rows), 256, 0, ctx->stream>>>(
        csr->range_offsets, csr->ranges, csr->single_offsets, csr->singles, csr->offsets, csr->rows,
        csr->indices);
    LO_CHECK_LAUNCH();
}

void free_csr_buffers(lo_context* ctx, lo_csr* csr) {
    if (csr->copied) {
        if (cudaEventQuery(csr->copied) != cudaSuccess) {
            // an async download still reads some buffers: release those once it has finished
            cudaGetLastError();
            lo_context::Deferred d{csr->copied, {}};
            void** bufs[4] = {reinterpret_cast<void**>(&csr->counts), reinterpret_cast<void**>(&csr->fps),
                              reinterpret_cast<void**>(&csr->offsets), reinterpret_cast<void**>(&csr->indices)};
            for (int b = 0; b < 4; ++b)
                if ((csr->copy_mask >> b) & 1u && *bufs[b]) {
                    d.ptrs.push_back(*bufs[b]);
                    *bufs[b] = nullptr;
                }
            ctx->deferred.push_back(std::move(d));
        } else {
            cudaEventDestroy(csr->copied);
        }
        csr->copied = nullptr;
        csr->copy_mask = 0;
    }
    dfree(ctx, csr->counts);
    dfree(ctx, csr->offsets);
    dfree(ctx, csr->indices);
    dfree(ctx, csr->fps);
    dfree(ctx, csr->range_offsets);
    dfree(ctx, csr->ranges);
    dfree(ctx, csr->single_offsets);
    dfree(ctx, csr->singles);
    csr->counts = nullptr, csr->offsets = nullptr, csr->indices = nullptr, csr->fps = nullptr;
    csr->range_offsets = nullptr, csr->ranges = nullptr, csr->single_offsets = nullptr;
    csr->singles = nullptr;
}

}  // namespace lo
