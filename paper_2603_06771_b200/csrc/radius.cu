// radius.cu -- K6 fixed-radius search (count -> u64 scan -> fill) and K8 row digests.
//
// Replaces neighbours_lin / neighbours_prune / run_radius_batch (search.cpp:45-156,
// :261-351).  One warp owns a tile of 32 consecutive queries (SFC-contiguous in Full mode)
// and walks the octree once for all of them: a node is entered while any lane's query
// intersects its box; a lane whose query contains the whole node emits the node's index
// range at once (the Keller-style prune of neighbours_prune) and ignores its descendants;
// leaf points are staged in shared memory and tested by every intersecting lane with the
// exact predicate.  DFS visits children in code order, so rows come out ascending like the
// reference's.
#include <chrono>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "radius_pt.cuh"

namespace lo {


template <int SHAPE, bool FILL>
__global__ void __launch_bounds__(kRadiusThreads) radius_kernel(
    const TNode* __restrict__ tn, const double* __restrict__ px, const double* __restrict__ py,
    const double* __restrict__ pz, Queries q, double r, double r2, u32* __restrict__ counts,
    const u64* __restrict__ offsets, u32* __restrict__ out) {
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
        u32 count = 0;
        u32* row = nullptr;
        if (FILL && active) row = out + offsets[qi];
        u32 skip_end = 0;
        int sp = 1;
        if (lane == 0) stack[0] = 0;
        __syncwarp();
        while (sp > 0) {
            const u32 t = stack[--sp];
            const NodeView nd = load_node(tn, t);
            int rel = kDisjoint;
            if (active && nd.begin >= skip_end) rel = relation<SHAPE>(cx, cy, cz, r, r2, nd);
            if (rel == kContains) {
                if (FILL)
                    for (u32 i = nd.begin; i < nd.end; ++i) row[count + (i - nd.begin)] = i;
                count += nd.end - nd.begin;
                skip_end = nd.end;
            }
            const unsigned hit = __ballot_sync(~0u, rel == kIntersects);
            if (!hit) continue;
            if (nd.nchild == 0) {
                for (u32 base = nd.begin; base < nd.end; base += 32) {
                    const u32 j = base + lane;
                    __syncwarp();
                    if (j < nd.end) {
                        sx[w][lane] = px[j];
                        sy[w][lane] = py[j];
                        sz[w][lane] = pz[j];
                    }
                    __syncwarp();
                    if (rel == kIntersects) {
                        const u32 cnt = min(32u, nd.end - base);
                        for (u32 jj = 0; jj < cnt; ++jj) {
                            if (contains<SHAPE>(cx, cy, cz, r, r2, sx[w][jj], sy[w][jj], sz[w][jj])) {
                                if (FILL) row[count] = base + jj;
                                ++count;
                            }
                        }
                    }
                }
            } else {
                __syncwarp();
                if (lane < static_cast<int>(nd.nchild)) stack[sp + nd.nchild - 1 - lane] = nd.child0 + lane;
                sp += nd.nchild;
                __syncwarp();
            }
        }
        if (!FILL && active) counts[qi] = count;
        __syncwarp();
    }
}

// K8: FNV-1a-64 per row over its indices (search.cpp:345-347).  The hash chain is sequential
// per row, so a thread owns a row; it reads the row with 16-byte loads (one L1 sector per load
// instead of one per index) after peeling to 16-byte alignment.
template <bool SMALL>
__global__ void radius_digest(const u64* __restrict__ offsets, const u32* __restrict__ idx, u64 m,
                              u64* __restrict__ fps) {
    for (u64 r = blockIdx.x * (u64)blockDim.x + threadIdx.x; r < m;
         r += (u64)gridDim.x * blockDim.x) {
        auto fnv = [](u64 h, u32 v) { return SMALL ? fnv_u24(h, v) : fnv_u32(h, v); };
        u64 h = kFnvOffset;
        u64 j = offsets[r];
        const u64 e = offsets[r + 1];
        for (; j < e && (j & 3); ++j) h = fnv(h, __ldg(idx + j));
        for (; j + 8 <= e; j += 8) {  // two loads in flight per iteration
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(idx + j));
            const uint4 u = __ldg(reinterpret_cast<const uint4*>(idx + j + 4));
            h = fnv(h, v.x);
            h = fnv(h, v.y);
            h = fnv(h, v.z);
            h = fnv(h, v.w);
            h = fnv(h, u.x);
            h = fnv(h, u.y);
            h = fnv(h, u.z);
            h = fnv(h, u.w);
        }
        if (j + 4 <= e) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(idx + j));
            h = fnv(h, v.x);
            h = fnv(h, v.y);
            h = fnv(h, v.z);
            h = fnv(h, v.w);
            j += 4;
        }
        for (; j < e; ++j) h = fnv(h, __ldg(idx + j));
        fps[r] = h;
    }
}

struct RecArgs {  // count-pass records for the replay fill (radius_pt.cuh)
    RecPool rp;
    const u32* list = nullptr;  // fill fallback: only these tiles
    u64 list_n = 0;
};

static bool float_path(const lo_octree* t, const lo_coded* c, const Queries& q, double r) {
    return make_float_test(r, std::max(c->bmax, q.bmax)).enabled && q.f && t->tf && c->pf && !force_fp64();
}


// fps != nullptr (count pass on the FP32 path): the row digests are computed by the count
// kernel itself (radius_pt_kernel<..., DIGEST>); returns whether it did.
template <bool FILL>
static bool launch_radius(lo_context* ctx, int shape, const lo_octree* t, const lo_coded* c,
                          const Queries& q, double r, u32* counts, const u64* offsets, u32* out,
                          const RecArgs& ra = RecArgs{}, u64* fps = nullptr) {
    const double r2 = r * r;  // SearchKernel ctor (geometry.hpp:107)
    const u64 tiles = ra.list ? ra.list_n : (q.m + 31) / 32;
    const int blocks = static_cast<int>(std::max<u64>(1, std::min<u64>((tiles + kRadiusWarps - 1) / kRadiusWarps,
                                                                      static_cast<u64>(ctx->sm_count) * 64)));
    if (float_path(t, c, q, r)) {
        FloatTest ft = make_float_test(r, std::max(c->bmax, q.bmax));
        // internal nodes of <= 256 points are taken whole: fewer node visits, and the walk's
        // per-point tile-box prefilter drops the far points of a whole node before they take
        // buffer slots.  With the prefilter, 256 beats 64 (cfg3 count 33.3 -> 30.2 ms, cfg1 r = 3
        // 4.95 -> 4.34 ms; 512: 30.5 / 4.37, 1024: 31.8 / 4.75; profiles/r2b/walk_knobs*.log).
        // Before the prefilter 64 was best (cfg1 count r = 3: 6.13 -> 5.04 ms vs 0).  LO_COARSE
        // overrides.
        static const u32 coarse = [] {
            const char* e = std::getenv("LO_COARSE");
            return e ? static_cast<u32>(std::strtoul(e, nullptr, 10)) : 256u;
        }();
        ft.coarse = coarse;
        // an 8-query group is tested against a child through its FP32 bounding box when its extent
        // is <= compact, else query by query (the box test cannot explode on tiles that straddle
        // an SFC jump).  cfg1 count: 4r 1.84 / 2.11 ms at r = 0.5 / 1, 8r 1.73 / 2.08, 16r 1.70 /
        // 2.08 but r = 3 5.15 vs 5.08 ms; unbounded: 16 ms at r = 1.  LO_COMPACT_MUL overrides.
        static const double compact_mul = [] {
            const char* e = std::getenv("LO_COMPACT_MUL");
            return e ? std::strtod(e, nullptr) : 8.0;
        }();
        const float compact = static_cast<float>(compact_mul * r);
        u64* counter = dalloc_t<u64>(ctx, 1);
        LO_CUDA(cudaMemsetAsync(counter, 0, 8, ctx->stream));
        const int pblocks = static_cast<int>(std::max<u64>(
            1, std::min<u64>((tiles + kPtWarps - 1) / kPtWarps, static_cast<u64>(ctx->sm_count) * LO_PT_MINB)));
        const int digest = FILL || !fps ? 0 : (c->n <= (1u << 24) ? 2 : 1);
#define LO_RADIUS_F(S)                                                                          \
    case S:                                                                                     \
        if (digest == 2)                                                                        \
            radius_pt_kernel<S, FILL, 2><<<pblocks, kPtThreads, 0, ctx->stream>>>(              \
                t->tf, c->pf, c->x, c->y, c->z, q, ft, compact, r, r2, counts, offsets, out,    \
                counter, ra.rp, ra.list, ra.list_n, fps);                                       \
        else if (digest == 1)                                                                   \
            radius_pt_kernel<S, FILL, 1><<<pblocks, kPtThreads, 0, ctx->stream>>>(              \
                t->tf, c->pf, c->x, c->y, c->z, q, ft, compact, r, r2, counts, offsets, out,    \
                counter, ra.rp, ra.list, ra.list_n, fps);                                       \
        else                                                                                    \
            radius_pt_kernel<S, FILL, 0><<<pblocks, kPtThreads, 0, ctx->stream>>>(              \
                t->tf, c->pf, c->x, c->y, c->z, q, ft, compact, r, r2, counts, offsets, out,    \
                counter, ra.rp, ra.list, ra.list_n, nullptr);                                   \
        break;
        switch (shape) {
            LO_RADIUS_F(LO_SPHERE)
            LO_RADIUS_F(LO_CIRCLE)
            LO_RADIUS_F(LO_CUBE)
            LO_RADIUS_F(LO_SQUARE)
            default: throw Error(LO_INVALID_ARGUMENT, "unknown kernel shape");
        }
#undef LO_RADIUS_F
        LO_CHECK_LAUNCH();
        dfree(ctx, counter);
        return digest != 0;
    }
    require(ra.list == nullptr, LO_LOGIC_ERROR, "tile-list fill needs the FP32 path");
#define LO_RADIUS_CASE(S)                                                                        \
    case S:                                                                                      \
        radius_kernel<S, FILL><<<blocks, kRadiusThreads, 0, ctx->stream>>>(t->tn, c->x, c->y,    \
                                                                           c->z, q, r, r2,       \
                                                                           counts, offsets, out); \
        break;
    switch (shape) {
        LO_RADIUS_CASE(LO_SPHERE)
        LO_RADIUS_CASE(LO_CIRCLE)
        LO_RADIUS_CASE(LO_CUBE)
        LO_RADIUS_CASE(LO_SQUARE)
        default: throw Error(LO_INVALID_ARGUMENT, "unknown kernel shape");
    }
#undef LO_RADIUS_CASE
    LO_CHECK_LAUNCH();
    return false;
}


static lo_csr* radius_search(lo_context* ctx, const lo_octree* t, const lo_coded* c, int shape,
                             double r, const Queries& q, bool fingerprint) {
    require(t != nullptr && c != nullptr, LO_INVALID_ARGUMENT, "null tree or cloud");
    require(r > 0.0 && std::isfinite(r), LO_INVALID_ARGUMENT,
            "kernel radius must be positive and finite");
    require(shape >= LO_SPHERE && shape <= LO_SQUARE, LO_INVALID_ARGUMENT, "unknown kernel shape");
    auto* out = new lo_csr;
    out->ctx = ctx;
    out->rows = q.m;
    cudaEvent_t e0, e1;
    {
        SlowLog slow("radius event create", 0);
        LO_CUDA(cudaEventCreate(&e0));
        LO_CUDA(cudaEventCreate(&e1));
    }
    RecArgs ra;
    u32* ovf = nullptr;
    u32* ovf_n = nullptr;
    // LO_DEBUG_HOST=1: host time of each segment of the call, printed for slow calls (diagnostic)
    static const bool dbg_host = std::getenv("LO_DEBUG_HOST") != nullptr;
    using clk = std::chrono::steady_clock;
    clk::time_point tm[8];
    int ntm = 0;
    const auto mark = [&] { if (dbg_host) tm[ntm++] = clk::now(); };
    try {
        mark();
        {
            SlowLog slow("radius events", 0);
            LO_CUDA(cudaEventRecord(e0, ctx->stream));
        }
        out->counts = big_alloc_t<u32>(ctx, q.m, &out->cap[0]);
        out->offsets = big_alloc_t<u64>(ctx, q.m + 1, &out->cap[2]);
        const u64 tiles = (q.m + 31) / 32;
        const bool no_fuse = env_flag("LO_RADIUS_NO_FUSE");
        const u32 cap = rec_cap();
        if (q.m && !no_fuse && float_path(t, c, q, r)) {
            try {
                RecSetup rs = setup_records(ctx, tiles, cap);
                ra.rp = rs.rp;
                ovf = rs.ovf;
                ovf_n = rs.ovf_n;
            } catch (const Error&) {  // not enough memory for the records: two-walk path
                ra = RecArgs{};
                ovf = ovf_n = nullptr;
            }
        }
        // LO_DIGEST_FUSED=1: the row digests ride along the count pass (radius_pt_kernel<..., DIGEST>).
        // Off by default: hashing each buffer's members per lane diverges with the members per row
        // (cfg3 count 40.4 -> 62.5 ms, cfg1 r = 3 5.1 -> 10.4 ms) and costs more than the separate
        // radius_digest pass it saves (9.2 ms at cfg3).
        if (fingerprint) out->fps = big_alloc_t<u64>(ctx, q.m, &out->cap[1]);
        u64* fused_fps = fingerprint && env_flag("LO_DIGEST_FUSED") ? out->fps : nullptr;
        stage_begin(ctx, "radius_count");
        bool digested = false;
        mark();
        if (q.m) digested = launch_radius<false>(ctx, shape, t, c, q, r, out->counts, nullptr, nullptr, ra, fused_fps);
        stage_end(ctx);
        stage_begin(ctx, "radius_scan");
        exclusive_scan_u32_to_u64(ctx, out->counts, out->offsets, q.m);
        stage_end(ctx);
        mark();
        out->total = read_scalar(ctx, out->offsets + q.m);
        mark();
        out->indices = big_alloc_t<u32>(ctx, out->total, &out->cap[3]);
        mark();
        stage_begin(ctx, "radius_fill");
        if (q.m && ra.rp.pool) {
            const u32 n_ovf = replay_records(ctx, RecSetup{ra.rp, ovf, ovf_n}, q.m, out->offsets,
                                             out->indices, out->total);
            static const bool debug = std::getenv("LO_DEBUG") != nullptr;
            if (debug)
                std::fprintf(stderr, "[lo] radius r=%g: %u of %llu tiles overflowed the %u-buffer records\n",
                             r, n_ovf, static_cast<unsigned long long>(tiles), cap);
            if (n_ovf) {
                RecArgs fb;
                fb.list = ovf;
                fb.list_n = n_ovf;
                launch_radius<true>(ctx, shape, t, c, q, r, nullptr, out->offsets, out->indices, fb);
            }
        } else if (q.m) {
            launch_radius<true>(ctx, shape, t, c, q, r, nullptr, out->offsets, out->indices);
        }
        stage_end(ctx);
        ra = RecArgs{};
        ovf = ovf_n = nullptr;
        LO_CUDA(cudaEventRecord(e1, ctx->stream));
        if (fingerprint && !digested) {
            // LO_DIGEST_AUX=1: the digests trail on the aux stream, overlapping the caller's next
            // batch.  Off by default: with the count kernels issue-bound, the overlap cost more than
            // it hid (cfg1 e2e 28.6 ms with it, 28.2 ms inline).
            const bool aux_digest = env_flag("LO_DIGEST_AUX");
            if (q.m && !ctx->timing && aux_digest) {
                // the digests trail on the aux stream while the caller's next batch counts;
                // readers of fps / indices (downloads, unsort, release) order behind `digested`
                LO_CUDA(cudaStreamWaitEvent(ctx->aux_stream, e1, 0));
                LO_CUDA(cudaEventCreateWithFlags(&out->digested, cudaEventDisableTiming));
                if (c->n <= (1u << 24))
                    radius_digest<true><<<std::max(1, ceil_div(q.m, 256)), 256, 0, ctx->aux_stream>>>(
                        out->offsets, out->indices, q.m, out->fps);
                else
                    radius_digest<false><<<std::max(1, ceil_div(q.m, 256)), 256, 0, ctx->aux_stream>>>(
                        out->offsets, out->indices, q.m, out->fps);
                LO_CHECK_LAUNCH();
                LO_CUDA(cudaEventRecord(out->digested, ctx->aux_stream));
            } else {
                stage_begin(ctx, "radius_digest");
                if (q.m)
                    (c->n <= (1u << 24) ? radius_digest<true> : radius_digest<false>)
                        <<<std::max(1, ceil_div(q.m, 256)), 256, 0, ctx->stream>>>(out->offsets, out->indices, q.m,
                                                                                   out->fps);
                LO_CHECK_LAUNCH();
                stage_end(ctx);
                LO_CUDA(cudaEventRecord(e1, ctx->stream));
            }
        }
        mark();
        spin_wait(e1);
        mark();
        LO_CUDA(cudaEventElapsedTime(&out->ms, e0, e1));
        if (dbg_host) {
            const double tot = std::chrono::duration<double, std::milli>(tm[ntm - 1] - tm[0]).count();
            {
                std::fprintf(stderr, "[lo] radius call %.2f ms host, %.2f ms device; segments:", tot, out->ms);
                for (int i = 1; i < ntm; ++i)
                    std::fprintf(stderr, " %.2f", std::chrono::duration<double, std::milli>(tm[i] - tm[i - 1]).count());
                std::fprintf(stderr, "\n");
            }
        }
        out->mean = q.m ? static_cast<double>(out->total) / static_cast<double>(q.m) : 0.0;
    } catch (...) {
        free_csr_buffers(ctx, out);
        delete out;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        throw;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return out;
}

// Centre indices from the host (or Full mode when null), validated against the cloud size.
u32* upload_centres(lo_context* ctx, const u32* centres_host, u64 m, u64 n) {
    if (!centres_host) return nullptr;
    for (u64 i = 0; i < m; ++i)
        require(centres_host[i] < n, LO_INVALID_ARGUMENT, "centre index out of range");
    u32* d = dalloc_t<u32>(ctx, m);
    LO_CUDA(cudaMemcpyAsync(d, centres_host, 4 * m, cudaMemcpyHostToDevice, ctx->stream));
    return d;
}

// Explicit query points (AoS host) -> SoA device, plus their FP32 filter copies relative to
// the cloud origin; *bmax bounds |query - origin| on every axis.
void upload_points(lo_context* ctx, const lo_coded* c, const double* xyz_host, u64 m, double** x,
                   double** y, double** z, float4** f, double* bmax) {
    std::vector<double> sx(m), sy(m), sz(m);
    std::vector<float4> sf(m);
    double b = 0.0;
    for (u64 i = 0; i < m; ++i) {
        sx[i] = xyz_host[3 * i];
        sy[i] = xyz_host[3 * i + 1];
        sz[i] = xyz_host[3 * i + 2];
        require(std::isfinite(sx[i]) && std::isfinite(sy[i]) && std::isfinite(sz[i]),
                LO_INVALID_ARGUMENT, "kernel center must be finite");
        const double rx = sx[i] - c->origin[0], ry = sy[i] - c->origin[1], rz = sz[i] - c->origin[2];
        sf[i] = make_float4(static_cast<float>(rx), static_cast<float>(ry), static_cast<float>(rz), 0.f);
        b = std::max({b, std::fabs(rx), std::fabs(ry), std::fabs(rz)});
    }
    *bmax = b * (1.0 + 1e-12);
    *x = dalloc_t<double>(ctx, m);
    *y = dalloc_t<double>(ctx, m);
    *z = dalloc_t<double>(ctx, m);
    *f = dalloc_t<float4>(ctx, m);
    LO_CUDA(cudaMemcpyAsync(*x, sx.data(), 8 * m, cudaMemcpyHostToDevice, ctx->stream));
    LO_CUDA(cudaMemcpyAsync(*y, sy.data(), 8 * m, cudaMemcpyHostToDevice, ctx->stream));
    LO_CUDA(cudaMemcpyAsync(*z, sz.data(), 8 * m, cudaMemcpyHostToDevice, ctx->stream));
    LO_CUDA(cudaMemcpyAsync(*f, sf.data(), 16 * m, cudaMemcpyHostToDevice, ctx->stream));
    sync(ctx);
}

}  // namespace lo

using namespace lo;

extern "C" {

int lo_radius(lo_context* ctx, const lo_octree* tree, const lo_coded* coded, int method, int shape,
              double radius, const uint32_t* centres_host, uint64_t m, int fingerprint,
              lo_csr** out) {
    return api_ctx(ctx, [&] {
        require(method != LO_METHOD_PTR, LO_INVALID_ARGUMENT,
                "run_radius_batch: ptr method needs a pointer octree");
        require(method == LO_METHOD_LIN || method == LO_METHOD_PRUNE || method == LO_METHOD_STRUCT,
                LO_INVALID_ARGUMENT, "unknown radius method");
        require(tree && coded, LO_INVALID_ARGUMENT, "null tree or cloud");
        const u64 rows = centres_host ? m : coded->n;
        ensure_float_shadows(ctx, coded, tree);
        u32* cidx = upload_centres(ctx, centres_host, m, coded->n);
        // explicit centres are searched in curve order, rows scattered back (centres.cu)
        // explicit centres are searched in curve order and the rows scattered back (centres.cu),
        // unless the caller asked for its own order (lo_context_set_option LO_OPT_CENTRE_ORDER = 0)
        const bool sorted = centres_host && ctx->centre_sort;
        SortedCentres sc = sort_centres(ctx, cidx, sorted ? m : 0);
        Queries q{coded->x, coded->y, coded->z, centres_host ? (sorted ? sc.idx : cidx) : nullptr, rows, coded->pf,
                  coded->bmax};
        try {
            *out = method == LO_METHOD_STRUCT
                       ? radius_struct_search(ctx, tree, coded, shape, radius, q, fingerprint != 0)
                       : radius_search(ctx, tree, coded, shape, radius, q, fingerprint != 0);
            if (sorted) unsort_csr(ctx, sc, *out);
        } catch (...) {
            dfree(ctx, cidx), dfree(ctx, sc.idx), dfree(ctx, sc.pos);
            throw;
        }
        dfree(ctx, cidx), dfree(ctx, sc.idx), dfree(ctx, sc.pos);
    });
}

int lo_radius_points(lo_context* ctx, const lo_octree* tree, const lo_coded* coded, int shape,
                     double radius, const double* queries_host, uint64_t m, lo_csr** out) {
    return api_ctx(ctx, [&] {
        require(tree && coded, LO_INVALID_ARGUMENT, "null tree or cloud");
        ensure_float_shadows(ctx, coded, tree);
        double *x = nullptr, *y = nullptr, *z = nullptr, bmax = 0.0;
        float4* f = nullptr;
        if (m) upload_points(ctx, coded, queries_host, m, &x, &y, &z, &f, &bmax);
        SortedCentres sc;
        try {
            // search in curve order (warp tiles of spatial neighbours), rows scattered back
            sc.pos = sort_points_sfc(ctx, coded, x, y, z, m);
            gather_queries(ctx, sc.pos, m, x, y, z, f);
            Queries q{x, y, z, nullptr, m, f, bmax};
            *out = radius_search(ctx, tree, coded, shape, radius, q, true);
            unsort_csr(ctx, sc, *out);
        } catch (...) {
            dfree(ctx, x), dfree(ctx, y), dfree(ctx, z), dfree(ctx, f), dfree(ctx, sc.pos);
            throw;
        }
        dfree(ctx, x), dfree(ctx, y), dfree(ctx, z), dfree(ctx, f), dfree(ctx, sc.pos);
    });
}

int lo_radius_struct_points(lo_context* ctx, const lo_octree* tree, const lo_coded* coded, int shape,
                            double radius, const double* queries_host, uint64_t m, lo_csr** out) {
    return api_ctx(ctx, [&] {
        require(tree && coded, LO_INVALID_ARGUMENT, "null tree or cloud");
        double *x = nullptr, *y = nullptr, *z = nullptr, bmax = 0.0;
        float4* f = nullptr;
        if (m) upload_points(ctx, coded, queries_host, m, &x, &y, &z, &f, &bmax);
        SortedCentres sc;
        try {
            sc.pos = sort_points_sfc(ctx, coded, x, y, z, m);
            gather_queries(ctx, sc.pos, m, x, y, z, f);
            Queries q{x, y, z, nullptr, m, f, bmax};
            *out = radius_struct_search(ctx, tree, coded, shape, radius, q, true);
            unsort_csr(ctx, sc, *out);
        } catch (...) {
            dfree(ctx, x), dfree(ctx, y), dfree(ctx, z), dfree(ctx, f), dfree(ctx, sc.pos);
            throw;
        }
        dfree(ctx, x), dfree(ctx, y), dfree(ctx, z), dfree(ctx, f), dfree(ctx, sc.pos);
    });
}

int lo_radius_range(lo_context* ctx, const lo_octree* tree, const lo_coded* coded, int method,
                    int shape, double radius, uint64_t begin, uint64_t end, int fingerprint,
                    lo_csr** out) {
    return api_ctx(ctx, [&] {
        require(method == LO_METHOD_LIN || method == LO_METHOD_PRUNE || method == LO_METHOD_STRUCT,
                LO_INVALID_ARGUMENT, "unknown radius method");
        require(tree && coded, LO_INVALID_ARGUMENT, "null tree or cloud");
        require(begin <= end && end <= coded->n, LO_INVALID_ARGUMENT, "centre range out of bounds");
        ensure_float_shadows(ctx, coded, tree);
        Queries q{coded->x + begin, coded->y + begin, coded->z + begin, nullptr, end - begin,
                  coded->pf + begin, coded->bmax};
        *out = method == LO_METHOD_STRUCT
                   ? radius_struct_search(ctx, tree, coded, shape, radius, q, fingerprint != 0)
                   : radius_search(ctx, tree, coded, shape, radius, q, fingerprint != 0);
    });
}

int lo_csr_info_get(const lo_csr* csr, lo_csr_info* out) {
    return api([&] {
        out->rows = csr->rows;
        out->total = csr->total;
        out->mean_count = csr->mean;
        out->device_ms = csr->ms;
    });
}

int lo_csr_download(lo_context* ctx, const lo_csr* csr, uint32_t* counts_host,
                    uint64_t* fingerprints_host, uint64_t* offsets_host, uint32_t* indices_host) {
    return api_ctx(ctx, [&] {
        if (csr->digested) LO_CUDA(cudaStreamWaitEvent(ctx->stream, csr->digested, 0));
        if (counts_host && csr->rows)
            LO_CUDA(cudaMemcpyAsync(counts_host, csr->counts, 4 * csr->rows, cudaMemcpyDeviceToHost,
                                    ctx->stream));
        if (fingerprints_host && csr->rows) {
            require(csr->fps != nullptr, LO_INVALID_ARGUMENT, "fingerprints were not computed");
            LO_CUDA(cudaMemcpyAsync(fingerprints_host, csr->fps, 8 * csr->rows,
                                    cudaMemcpyDeviceToHost, ctx->stream));
        }
        if (offsets_host)
            LO_CUDA(cudaMemcpyAsync(offsets_host, csr->offsets, 8 * (csr->rows + 1),
                                    cudaMemcpyDeviceToHost, ctx->stream));
        if (indices_host && csr->total) {
            ensure_expanded(ctx, const_cast<lo_csr*>(csr));
            LO_CUDA(cudaMemcpyAsync(indices_host, csr->indices, 4 * csr->total,
                                    cudaMemcpyDeviceToHost, ctx->stream));
        }
        sync(ctx);
    });
}

int lo_csr_download_async(lo_context* ctx, lo_csr* csr, uint32_t* counts_host,
                          uint64_t* fingerprints_host, uint64_t* offsets_host, uint32_t* indices_host) {
    return api_ctx(ctx, [&] {
        require(csr != nullptr, LO_INVALID_ARGUMENT, "null result");
        require(!fingerprints_host || csr->fps, LO_INVALID_ARGUMENT, "fingerprints were not computed");
        if (indices_host && csr->total) ensure_expanded(ctx, csr);
        if (!csr->copied) LO_CUDA(cudaEventCreateWithFlags(&csr->copied, cudaEventDisableTiming));
        cudaEvent_t ready;
        LO_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
        LO_CUDA(cudaEventRecord(ready, ctx->stream));
        LO_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ready, 0));
        cudaEventDestroy(ready);  // released once the recorded work completes
        if (csr->digested) LO_CUDA(cudaStreamWaitEvent(ctx->copy_stream, csr->digested, 0));
        cudaStream_t s = ctx->copy_stream;
        csr->copy_mask |= (counts_host ? 1u : 0u) | (fingerprints_host ? 2u : 0u) | (offsets_host ? 4u : 0u) |
                          (indices_host ? 8u : 0u);
        if (counts_host && csr->rows)
            LO_CUDA(cudaMemcpyAsync(counts_host, csr->counts, 4 * csr->rows, cudaMemcpyDeviceToHost, s));
        if (fingerprints_host && csr->rows)
            LO_CUDA(cudaMemcpyAsync(fingerprints_host, csr->fps, 8 * csr->rows, cudaMemcpyDeviceToHost, s));
        if (offsets_host)
            LO_CUDA(cudaMemcpyAsync(offsets_host, csr->offsets, 8 * (csr->rows + 1), cudaMemcpyDeviceToHost, s));
        if (indices_host && csr->total)
            LO_CUDA(cudaMemcpyAsync(indices_host, csr->indices, 4 * csr->total, cudaMemcpyDeviceToHost, s));
        LO_CUDA(cudaEventRecord(csr->copied, s));
    });
}

int lo_csr_device_ptrs(const lo_csr* csr, const uint64_t** offsets, const uint32_t** indices) {
    if (!csr) return api([] { throw Error(LO_INVALID_ARGUMENT, "null result"); });
    return api_ctx(csr->ctx, [&] {
        if (indices) ensure_expanded(csr->ctx, const_cast<lo_csr*>(csr));
        if (offsets) *offsets = csr->offsets;
        if (indices) *indices = csr->indices;
    });
}

int lo_csr_struct_info(const lo_csr* csr, uint64_t* total_ranges, uint64_t* total_singles) {
    return api([&] {
        require(csr && csr->is_struct, LO_INVALID_ARGUMENT, "not a Struct radius result");
        if (total_ranges) *total_ranges = csr->total_ranges;
        if (total_singles) *total_singles = csr->total_singles;
    });
}

int lo_csr_struct_download(lo_context* ctx, const lo_csr* csr, uint64_t* range_offsets_host,
                           uint32_t* ranges_host, uint64_t* single_offsets_host,
                           uint32_t* singles_host) {
    return api_ctx(ctx, [&] {
        require(csr && csr->is_struct, LO_INVALID_ARGUMENT, "not a Struct radius result");
        if (range_offsets_host)
            LO_CUDA(cudaMemcpyAsync(range_offsets_host, csr->range_offsets, 8 * (csr->rows + 1),
                                    cudaMemcpyDeviceToHost, ctx->stream));
        if (ranges_host && csr->total_ranges)
            LO_CUDA(cudaMemcpyAsync(ranges_host, csr->ranges, 8 * csr->total_ranges,
                                    cudaMemcpyDeviceToHost, ctx->stream));
        if (single_offsets_host)
            LO_CUDA(cudaMemcpyAsync(single_offsets_host, csr->single_offsets, 8 * (csr->rows + 1),
                                    cudaMemcpyDeviceToHost, ctx->stream));
        if (singles_host && csr->total_singles)
            LO_CUDA(cudaMemcpyAsync(singles_host, csr->singles, 4 * csr->total_singles,
                                    cudaMemcpyDeviceToHost, ctx->stream));
        sync(ctx);
    });
}

int lo_csr_destroy(lo_csr* csr) {
    if (!csr) return LO_OK;
    return api_ctx(csr->ctx, [&] {
        free_csr_buffers(csr->ctx, csr);
        delete csr;
    });
}

}  // extern "C"
