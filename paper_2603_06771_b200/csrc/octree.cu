// octree.cu -- K5 parallel linear-octree build over the sorted codes.
//
// Replaces build_leaves + link_internal (linear_octree.cpp:23-137) with a scan-based build
// that produces byte-identical LeafArray and preorder InternalNode tables:
//
//  * A depth-d block is internal iff it holds more than n_max points and d < level
//    (linear_octree.cpp:44-49); all its ancestors then are too.
//  * Point i opens the internal node at depth d iff it is the block's first point,
//    cpl(code[i-1], code[i]) < d, and the block overflows, cpl(code[i], code[i+n_max]) >= d,
//    where cpl = common octal-prefix length.  Preorder (linear_octree.cpp:113-137) equals
//    the order (first point, depth), so an exclusive scan of per-point counts numbers the
//    internal nodes exactly as the reference's recursion does.
//  * Leaves are the non-internal children of internal nodes (empty ones included).  The
//    leaves before node k's block are 7*(k - depth) + (sum of the prefix's top octal
//    digits), so each node numbers its own leaf children without a global pass.
//
// The traversal side gets a second, children-contiguous table of non-empty nodes (TNode)
// with tight boxes built bottom-up (Karras-style arrival counters).
#include <algorithm>
#include <cmath>

#include "lo_internal.cuh"

namespace lo {

__device__ __forceinline__ int cpl_of(u64 a, u64 b, int level) {
    if (a == b) return level;
    return (__clzll(static_cast<long long>(a ^ b)) - (64 - 3 * level)) / 3;
}

__device__ __forceinline__ u32 lower_bound_dev(const u64* __restrict__ codes, u32 lo, u32 hi,
                                               u64 key) {
    while (lo < hi) {
        const u32 mid = lo + ((hi - lo) >> 1);
        if (codes[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ int first_open_depth(const u64* __restrict__ codes, u64 i, int level) {
    return i == 0 ? 0 : cpl_of(codes[i - 1], codes[i], level) + 1;
}

// number of internal nodes whose first point is i
__global__ void open_count(const u64* __restrict__ codes, u64 n, u32 n_max, int level,
                           u32* __restrict__ cnt) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n;
         i += (u64)gridDim.x * blockDim.x) {
        u32 c = 0;
        if (i + n_max < n && level > 0) {
            const int lo = first_open_depth(codes, i, level);
            const int hi = min(level - 1, cpl_of(codes[i], codes[i + n_max], level));
            c = hi >= lo ? static_cast<u32>(hi - lo + 1) : 0u;
        }
        cnt[i] = c;
    }
}

__global__ void open_emit(const u64* __restrict__ codes, u64 n, const u32* __restrict__ cnt,
                          const u32* __restrict__ S, int level, u32* __restrict__ npoint,
                          u8* __restrict__ ndepth) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n;
         i += (u64)gridDim.x * blockDim.x) {
        const u32 c = cnt[i];
        if (c == 0) continue;
        const int lo = first_open_depth(codes, i, level);
        const u32 base = S[i];
        for (u32 t = 0; t < c; ++t) {
            npoint[base + t] = static_cast<u32>(i);
            ndepth[base + t] = static_cast<u8>(lo + t);
        }
    }
}

// One thread per internal node: range, children, child mask, leaf children.
__global__ void link_nodes(const u64* __restrict__ codes, u32 n, u32 n_max, int level,
                           const u32* __restrict__ S, const u32* __restrict__ npoint,
                           const u8* __restrict__ ndepth, u32 internal,
                           lo_internal_node* __restrict__ nodes, u64* __restrict__ bounds,
                           u32* __restrict__ offsets, u32* __restrict__ nchild) {
    for (u64 k = blockIdx.x * (u64)blockDim.x + threadIdx.x; k < internal;
         k += (u64)gridDim.x * blockDim.x) {
        const u32 i = npoint[k];
        const int d = ndepth[k];
        const int shift = 3 * (level - d);
        const u64 span = 1ull << shift;
        const u64 prefix = d == 0 ? 0ull : (codes[i] >> shift) << shift;
        const u32 end = lower_bound_dev(codes, i, n, prefix + span);
        const u64 sub = span >> 3;
        u64 leaf = 7ull * (k - static_cast<u64>(d));
        for (int t = 1; t <= d; ++t) leaf += (prefix >> (3 * (level - t))) & 7u;
        u32 cb[9];
        cb[0] = i;
        cb[8] = end;
        for (int c = 1; c < 8; ++c) cb[c] = lower_bound_dev(codes, cb[c - 1], end, prefix + c * sub);
        lo_internal_node nd;
        nd.prefix = prefix;
        nd.begin = i;
        nd.end = end;
        nd.depth = static_cast<u8>(d);
        u8 mask = 0;
        for (int c = 0; c < 8; ++c) {
            const u32 count = cb[c + 1] - cb[c];
            if (count > n_max && d + 1 < level) {
                const u32 j = S[cb[c]] + static_cast<u32>(d + 1 - first_open_depth(codes, cb[c], level));
                nd.children[c] = static_cast<i32>(j);
                leaf += 1 + 7ull * (S[cb[c + 1]] - j);
            } else {
                nd.children[c] = ~static_cast<i32>(leaf);
                bounds[leaf] = prefix + c * sub;
                offsets[leaf] = cb[c];
                ++leaf;
            }
            if (count) mask |= static_cast<u8>(1u << c);
        }
        nd.child_mask = mask;
        for (int b = 0; b < 6; ++b) nd.pad_[b] = 0;
        nodes[k] = nd;
        nchild[k] = __popc(mask);
    }
}

__global__ void leaves_tail(u64* bounds, u32* offsets, u64 leaves, u64 full, u32 n) {
    bounds[leaves] = full;
    offsets[leaves] = n;
    if (leaves == 1) {  // single-leaf tree: root leaf covers everything
        bounds[0] = 0;
        offsets[0] = 0;
    }
}

// TNode table: root = 0; the non-empty children of internal node k sit at
// 1 + tbase[k] + rank, in code order.
__global__ void emit_tnodes(const lo_internal_node* __restrict__ nodes, u32 internal,
                            const u32* __restrict__ tbase, const u32* __restrict__ nchild,
                            const u32* __restrict__ offsets, TNode* __restrict__ tn,
                            u32* __restrict__ parent, u32* __restrict__ tid_of) {
    for (u64 k = blockIdx.x * (u64)blockDim.x + threadIdx.x; k < internal;
         k += (u64)gridDim.x * blockDim.x) {
        const lo_internal_node nd = nodes[k];
        u32 t = 1 + tbase[k];
        if (k == 0) {
            tn[0].begin = nd.begin;
            tn[0].end = nd.end;
            tn[0].child0 = 1 + tbase[0];
            tn[0].nchild = nchild[0];
            parent[0] = ~0u;
            tid_of[0] = 0;
        }
        for (int c = 0; c < 8; ++c) {
            if (!((nd.child_mask >> c) & 1)) continue;
            const i32 ch = nd.children[c];
            TNode& o = tn[t];
            if (ch >= 0) {
                const lo_internal_node& cn = nodes[ch];
                o.begin = cn.begin;
                o.end = cn.end;
                o.child0 = 1 + tbase[ch];
                o.nchild = nchild[ch];
                tid_of[ch] = t;
            } else {
                o.begin = offsets[~ch];
                o.end = offsets[~ch + 1];
                o.child0 = 0;
                o.nchild = 0;
            }
            parent[t] = static_cast<u32>(k);
            ++t;
        }
    }
}

__global__ void single_leaf_tnode(TNode* tn, u32 n, u32* parent) {
    tn[0].begin = 0;
    tn[0].end = n;
    tn[0].child0 = 0;
    tn[0].nchild = 0;
    parent[0] = ~0u;
}

// Leaf boxes from their points, then bottom-up unions: the last child to arrive at a parent
// (arrival counter) computes the parent's box and continues upward.
// Tight boxes bottom-up, in two launches.  tnode_leaf_boxes: a group of 8 lanes takes one leaf --
// coalesced loads of its points and a 3-step shuffle reduction (leaves hold ~13 points at cfg3; a
// thread per leaf left 4.5 of 32 lanes busy and read 32 scattered lines per load).
// tnode_boxes: a thread per leaf carries its box to the parents whose children have all arrived
// (arrival counters); a group leader doing that chain held its 7 lanes idle (12 ms vs 2.8 ms).
__global__ void __launch_bounds__(128) tnode_leaf_boxes(TNode* tn, u64 tnodes, const double* __restrict__ x,
                                                        const double* __restrict__ y,
                                                        const double* __restrict__ z) {
    const int sub = threadIdx.x & 7;
    const u64 groups = (static_cast<u64>(gridDim.x) * blockDim.x) >> 3;
    for (u64 t = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 3; t < tnodes; t += groups) {
        if (tn[t].nchild != 0) continue;  // group-uniform
        const u32 b = tn[t].begin, e = tn[t].end;
        double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (u32 i = b + sub; i < e; i += 8) {
            const double v[3] = {x[i], y[i], z[i]};
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                lo[a] = fmin(lo[a], v[a]);
                hi[a] = fmax(hi[a], v[a]);
            }
        }
        const unsigned gm = 0xffu << (threadIdx.x & 24);
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) {
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                lo[a] = fmin(lo[a], __shfl_xor_sync(gm, lo[a], o));
                hi[a] = fmax(hi[a], __shfl_xor_sync(gm, hi[a], o));
            }
        }
        if (sub < 3) {
            tn[t].lo[sub] = lo[sub];
            tn[t].hi[sub] = hi[sub];
        }
    }
}

__global__ void __launch_bounds__(128) tnode_boxes(TNode* tn, u64 tnodes, const u32* __restrict__ parent,
                                                   const u32* __restrict__ tid_of, u32* __restrict__ arrivals) {
    for (u64 t = blockIdx.x * (u64)blockDim.x + threadIdx.x; t < tnodes; t += (u64)gridDim.x * blockDim.x) {
        if (tn[t].nchild != 0) continue;
        u32 cur = parent[t];
        while (cur != ~0u) {
            __threadfence();
            if (atomicAdd(&arrivals[cur], 1u) + 1 != tn[tid_of[cur]].nchild) break;
            __threadfence();
            const u32 pt = tid_of[cur];
            const u32 c0 = __ldcg(&tn[pt].child0);
            const u32 nc = __ldcg(&tn[pt].nchild);
            double plo[3], phi[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                plo[a] = __ldcg(&tn[c0].lo[a]);
                phi[a] = __ldcg(&tn[c0].hi[a]);
            }
            for (u32 c = 1; c < nc; ++c) {
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    plo[a] = fmin(plo[a], __ldcg(&tn[c0 + c].lo[a]));
                    phi[a] = fmax(phi[a], __ldcg(&tn[c0 + c].hi[a]));
                }
            }
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                __stcg(&tn[pt].lo[a], plo[a]);
                __stcg(&tn[pt].hi[a], phi[a]);
            }
            cur = parent[pt];
        }
    }
}

// FP32 shadow of the traversal table: boxes relative to the cloud origin rounded outward
// (directed-rounding subtract, then directed-rounding narrowing), so they keep containing
// every point's exact relative position.
__global__ void tnode_float(const TNode* __restrict__ tn, u64 T, TNodeF* __restrict__ tf,
                            double ox, double oy, double oz) {
    for (u64 t = blockIdx.x * (u64)blockDim.x + threadIdx.x; t < T;
         t += (u64)gridDim.x * blockDim.x) {
        const TNode nd = tn[t];
        const double o[3] = {ox, oy, oz};
        float lo[3], hi[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            lo[a] = __double2float_rd(__dsub_rd(nd.lo[a], o[a]));
            hi[a] = __double2float_ru(__dsub_ru(nd.hi[a], o[a]));
        }
        TNodeF f;
        f.a = make_float4(lo[0], lo[1], lo[2], __uint_as_float(nd.begin));
        f.b = make_float4(hi[0], hi[1], hi[2], __uint_as_float(nd.end));
        f.c = make_uint4(nd.child0, nd.nchild, 0u, 0u);
        tf[t] = f;
    }
}

void build_float_points(lo_context* ctx, lo_coded* c);  // reorder.cu

static void build_float_nodes(lo_context* ctx, lo_octree* t, const lo_coded* c) {
    if (t->tf) return;
    t->tf = dalloc_t<TNodeF>(ctx, t->tnodes);
    const int g = static_cast<int>(std::max<u64>(1, std::min<u64>((t->tnodes + 255) / 256,
                                                                  ctx->sm_count * 16ull)));
    tnode_float<<<g, 256, 0, ctx->stream>>>(t->tn, t->tnodes, t->tf,
                                                                 c->origin[0], c->origin[1],
                                                                 c->origin[2]);
    LO_CHECK_LAUNCH();
}

// Lazily built device data is published complete: built under the handle's own mutex and
// synchronized before the lock is released, so another context sharing the (read-only) handle
// never sees a pointer whose kernels are still running on the builder's stream.
void ensure_float_shadows(lo_context* ctx, const lo_coded* coded, const lo_octree* tree) {
    auto* c = const_cast<lo_coded*>(coded);
    auto* t = const_cast<lo_octree*>(tree);
    {
        std::lock_guard<std::mutex> g(c->lazy_mu);
        if (!c->pf) {
            SlowLog slow("float points", c->n);
            build_float_points(ctx, c);
            sync(ctx);
        }
    }
    std::lock_guard<std::mutex> g(t->lazy_mu);
    if (!t->tf) {
        SlowLog slow("float nodes", 0);
        build_float_nodes(ctx, t, coded);
        sync(ctx);
    }
}

// node_bounds (linear_octree.cpp:139-147): padded octant box of a NodeRef.
struct BoundsParams {
    double box[6];
    int level;
    u8 dec[32 * 8];
};

__device__ __forceinline__ double pad_down(double v) { return dbl_from_order_key(dbl_order_key(v) - 2); }
__device__ __forceinline__ double pad_up(double v) { return dbl_from_order_key(dbl_order_key(v) + 2); }

// octant_bounds (sfc.cpp:110-127) of the block at `depth` starting at cell code `prefix`
// (prefix_to_octant_bounds, sfc.cpp:129-141): decode the top `depth` digits, scale, pad.
__device__ void octant_box(u64 prefix, int depth, const BoundsParams& p, double* o) {
    if (depth == 0) {
        for (int a = 0; a < 6; ++a) o[a] = p.box[a];
        return;
    }
    const u64 top = prefix >> (3 * (p.level - depth));
    u32 h[3] = {0, 0, 0}, s = 0;
    for (int d = depth - 1; d >= 0; --d) {
        const u32 e = p.dec[s * 8 + ((top >> (3 * d)) & 7u)];
        h[0] = h[0] << 1 | ((e >> 2) & 1u);
        h[1] = h[1] << 1 | ((e >> 1) & 1u);
        h[2] = h[2] << 1 | (e & 1u);
        s = e >> 3;
    }
    const double inv = ldexp(1.0, -depth);
    for (int a = 0; a < 3; ++a) {
        const double side = (p.box[3 + a] - p.box[a]) * inv;
        const double lo = p.box[a] + static_cast<double>(h[a]) * side;
        const double hi = lo + side;
        o[a] = pad_down(lo);
        o[3 + a] = pad_up(hi);
    }
}

__global__ void node_bounds_kernel(const i32* __restrict__ refs, u64 count,
                                   const lo_internal_node* __restrict__ nodes,
                                   const u64* __restrict__ bounds, BoundsParams p,
                                   double* __restrict__ out) {
    for (u64 r = blockIdx.x * (u64)blockDim.x + threadIdx.x; r < count;
         r += (u64)gridDim.x * blockDim.x) {
        const i32 ref = refs[r];
        u64 prefix;
        int depth;
        if (ref < 0) {
            const u32 id = static_cast<u32>(~ref);
            prefix = bounds[id];
            const u64 span = bounds[id + 1] - bounds[id];
            depth = p.level - (__ffsll(static_cast<long long>(span)) - 1) / 3;
        } else {
            prefix = nodes[ref].prefix;
            depth = nodes[ref].depth;
        }
        octant_box(prefix, depth, p, out + 6 * r);
    }
}

// Depth of every traversal node, one level per launch (children are one level below).
__global__ void tnode_depth_step(const TNode* __restrict__ tn, u64 count, u8* __restrict__ depth,
                                 int d) {
    for (u64 t = blockIdx.x * (u64)blockDim.x + threadIdx.x; t < count;
         t += (u64)gridDim.x * blockDim.x) {
        if (depth[t] != d) continue;
        const u32 c0 = tn[t].child0, nc = tn[t].nchild;
        for (u32 j = 0; j < nc; ++j) depth[c0 + j] = static_cast<u8>(d + 1);
    }
}

// Padded octant box of every traversal node: the block at its depth holding its first point.
__global__ void tnode_ref_boxes(const TNode* __restrict__ tn, const u8* __restrict__ depth, u64 count,
                                const u64* __restrict__ codes, BoundsParams p, double* __restrict__ rb) {
    for (u64 t = blockIdx.x * (u64)blockDim.x + threadIdx.x; t < count;
         t += (u64)gridDim.x * blockDim.x) {
        const int d = depth[t];
        const u64 code = codes[tn[t].begin];
        const u64 prefix = d == 0 ? 0ull : code & ~((1ull << (3 * (p.level - d))) - 1ull);
        octant_box(prefix, d, p, rb + 6 * t);
    }
}

// FP32 copies of the reference boxes for the filtered Struct relation: outward-rounded, relative
// to the cloud origin like the point filter copies.
__global__ void ref_boxes_float(const double* __restrict__ rb, u64 count, double ox, double oy, double oz,
                                float4* __restrict__ rbf) {
    for (u64 t = blockIdx.x * (u64)blockDim.x + threadIdx.x; t < count; t += (u64)gridDim.x * blockDim.x) {
        const double* b = rb + 6 * t;
        const double o[3] = {ox, oy, oz};
        float lo[3], hi[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            lo[a] = __double2float_rd(__dsub_rd(b[a], o[a]));
            hi[a] = __double2float_ru(__dsub_ru(b[3 + a], o[a]));
        }
        rbf[2 * t] = make_float4(lo[0], lo[1], lo[2], 0.f);
        rbf[2 * t + 1] = make_float4(hi[0], hi[1], hi[2], 0.f);
    }
}

void ensure_ref_boxes(lo_context* ctx, const lo_coded* coded, const lo_octree* tree) {
    auto* t = const_cast<lo_octree*>(tree);
    std::lock_guard<std::mutex> g(t->lazy_mu);  // published complete (see ensure_float_shadows)
    if (t->rb && t->rbf) return;
    const u64 T = t->tnodes;
    u8* depth = dalloc_t<u8>(ctx, T);
    double* rb = nullptr;
    try {
        rb = dalloc_t<double>(ctx, 6 * T);
        LO_CUDA(cudaMemsetAsync(depth, 0xff, T, ctx->stream));
        LO_CUDA(cudaMemsetAsync(depth, 0, 1, ctx->stream));
        const int g = static_cast<int>(std::max<u64>(1, std::min<u64>((T + 255) / 256, ctx->sm_count * 16ull)));
        for (int d = 0; d < t->level; ++d) {
            tnode_depth_step<<<g, 256, 0, ctx->stream>>>(t->tn, T, depth, d);
            LO_CHECK_LAUNCH();
        }
        BoundsParams p;
        std::memcpy(p.box, t->disc_box, sizeof p.box);
        p.level = t->level;
        std::memcpy(p.dec, curve_tables(t->curve).dec, sizeof p.dec);
        tnode_ref_boxes<<<g, 256, 0, ctx->stream>>>(t->tn, depth, T, coded->codes, p, rb);
        LO_CHECK_LAUNCH();
        t->rbf = dalloc_t<float4>(ctx, 2 * T);
        ref_boxes_float<<<g, 256, 0, ctx->stream>>>(rb, T, coded->origin[0], coded->origin[1], coded->origin[2],
                                                    t->rbf);
        LO_CHECK_LAUNCH();
    } catch (...) {
        dfree(ctx, depth);
        dfree(ctx, rb);
        dfree(ctx, t->rbf);
        t->rbf = nullptr;
        throw;
    }
    dfree(ctx, depth);
    sync(ctx);
    t->rb = rb;
}

__global__ void check_sorted(const u64* __restrict__ codes, u64 n, u64 full, u32* __restrict__ flags) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n;
         i += (u64)gridDim.x * blockDim.x) {
        if (i > 0 && codes[i - 1] > codes[i]) atomicOr(flags, 1u);
        if (codes[i] >= full) atomicOr(flags, 2u);
    }
}

static int grid1(lo_context* ctx, u64 n, int threads = 256) {
    const u64 want = (n + threads - 1) / threads;
    return static_cast<int>(std::max<u64>(1, std::min<u64>(want, static_cast<u64>(ctx->sm_count) * 16)));
}

struct LeafBuild {
    u64 internal = 0, leaves = 0;
    u64* bounds = nullptr;
    u32* offsets = nullptr;
    lo_internal_node* nodes = nullptr;
    u32* nchild = nullptr;
    int max_depth = 0;
};

// Internal-node table + LeafArray for sorted device codes.
static LeafBuild build_tables(lo_context* ctx, const u64* codes, u64 n, u32 n_max, int level) {
    LeafBuild r;
    u32* cnt = dalloc_t<u32>(ctx, n);
    u32* S = dalloc_t<u32>(ctx, n + 1);
    open_count<<<grid1(ctx, n), 256, 0, ctx->stream>>>(codes, n, n_max, level, cnt);
    LO_CHECK_LAUNCH();
    exclusive_scan_u32(ctx, cnt, S, n);
    const u32 I = read_scalar(ctx, S + n);
    r.internal = I;
    r.leaves = 7ull * I + 1;
    r.bounds = dalloc_t<u64>(ctx, r.leaves + 1);
    r.offsets = dalloc_t<u32>(ctx, r.leaves + 1);
    r.nodes = dalloc_t<lo_internal_node>(ctx, I);
    r.nchild = dalloc_t<u32>(ctx, I + 1);
    if (I > 0) {
        u32* npoint = dalloc_t<u32>(ctx, I);
        u8* ndepth = dalloc_t<u8>(ctx, I);
        open_emit<<<grid1(ctx, n), 256, 0, ctx->stream>>>(codes, n, cnt, S, level, npoint, ndepth);
        LO_CHECK_LAUNCH();
        link_nodes<<<grid1(ctx, I, 128), 128, 0, ctx->stream>>>(
            codes, static_cast<u32>(n), n_max, level, S, npoint, ndepth, I, r.nodes, r.bounds,
            r.offsets, r.nchild);
        LO_CHECK_LAUNCH();
        dfree(ctx, npoint);
        dfree(ctx, ndepth);
    }
    const u64 full = 1ull << (3 * level);
    leaves_tail<<<1, 1, 0, ctx->stream>>>(r.bounds, r.offsets, r.leaves, full, static_cast<u32>(n));
    LO_CHECK_LAUNCH();
    dfree(ctx, cnt);
    dfree(ctx, S);
    return r;
}

static void validate_codes(lo_context* ctx, const u64* codes, u64 n, int level) {
    u32* flags = dalloc_t<u32>(ctx, 1);
    LO_CUDA(cudaMemsetAsync(flags, 0, 4, ctx->stream));
    check_sorted<<<grid1(ctx, n), 256, 0, ctx->stream>>>(codes, n, 1ull << (3 * level), flags);
    LO_CHECK_LAUNCH();
    const u32 f = read_scalar(ctx, flags);
    dfree(ctx, flags);
    require(!(f & 1u), LO_INVALID_ARGUMENT, "build_leaves: codes are not sorted");
    require(!(f & 2u), LO_INVALID_ARGUMENT, "build_leaves: code exceeds 8^level");
}

// Traversal table, tight boxes and FP32 shadow over a finished LeafBuild; takes ownership of
// lb's buffers.
static lo_octree* finish_octree(lo_context* ctx, const lo_coded* coded, LeafBuild& lb, u32 n_max,
                                int level, int curve, const double disc_box[6]) {
    const u64 n = coded->n;
    auto* t = new lo_octree;
    t->ctx = ctx;
    t->coded = coded;
    t->points = n;
    t->leaves = lb.leaves;
    t->internal = lb.internal;
    t->root = lb.internal > 0 ? 0 : ~0;
    t->n_max = n_max;
    t->level = level;
    t->curve = curve;
    std::memcpy(t->disc_box, disc_box, sizeof t->disc_box);
    t->bounds = lb.bounds;
    t->offsets = lb.offsets;
    t->nodes = lb.nodes;
    const u32 I = static_cast<u32>(lb.internal);
    // traversal table
    u32* tbase = dalloc_t<u32>(ctx, I + 1);
    u64 T = 1;
    if (I > 0) {
        exclusive_scan_u32(ctx, lb.nchild, tbase, I);
        T = 1 + read_scalar(ctx, tbase + I);
    }
    t->tnodes = T;
    t->tn = dalloc_t<TNode>(ctx, T);
    u32* parent = dalloc_t<u32>(ctx, T);
    u32* tid_of = dalloc_t<u32>(ctx, I + 1);
    u32* arrivals = dalloc_t<u32>(ctx, I + 1);
    LO_CUDA(cudaMemsetAsync(arrivals, 0, 4ull * (I + 1), ctx->stream));
    if (I > 0) {
        emit_tnodes<<<grid1(ctx, I, 128), 128, 0, ctx->stream>>>(lb.nodes, I, tbase, lb.nchild,
                                                                 lb.offsets, t->tn, parent, tid_of);
    } else {
        single_leaf_tnode<<<1, 1, 0, ctx->stream>>>(t->tn, static_cast<u32>(n), parent);
    }
    LO_CHECK_LAUNCH();
    tnode_leaf_boxes<<<grid1(ctx, 8 * T, 128), 128, 0, ctx->stream>>>(t->tn, T, coded->x, coded->y, coded->z);
    LO_CHECK_LAUNCH();
    tnode_boxes<<<grid1(ctx, T, 128), 128, 0, ctx->stream>>>(t->tn, T, parent, tid_of, arrivals);
    LO_CHECK_LAUNCH();
    build_float_nodes(ctx, t, coded);
    dfree(ctx, tbase);
    dfree(ctx, parent);
    dfree(ctx, tid_of);
    dfree(ctx, arrivals);
    dfree(ctx, lb.nchild);
    lb = LeafBuild{};
    sync(ctx);
    return t;
}

static lo_octree* octree_build(lo_context* ctx, const lo_coded* coded, u32 n_max) {
    require(coded != nullptr, LO_INVALID_ARGUMENT, "null coded cloud");
    require(n_max >= 1, LO_INVALID_ARGUMENT, "build_leaves: n_max must be >= 1");
    stage_begin(ctx, "build");
    LeafBuild lb = build_tables(ctx, coded->codes, coded->n, n_max, coded->level);
    lo_octree* t = finish_octree(ctx, coded, lb, n_max, coded->level, coded->curve, coded->disc_box);
    stage_end(ctx);
    return t;
}

// ---- LinearOctree(LeafArray, Discretizer, Curve, n_max) (linear_octree.cpp:84-137) ------
// link_range's recursion, without recursion: leaf i starts the internal blocks at the depths d
// < depth(leaf i) at which its start b[i] is block-aligned, and preorder == (first leaf,
// depth), so a scan of the per-leaf counts numbers the nodes like link_range does.
__device__ __forceinline__ int leaf_depth(u64 span, int level) {
    return level - (__ffsll(static_cast<long long>(span)) - 1) / 3;
}
__device__ __forceinline__ int first_open_depth(u64 start, int level) {
    if (start == 0) return 0;
    const int tz = (__ffsll(static_cast<long long>(start)) - 1) / 3;  // trailing zero octal digits
    return tz >= level ? 0 : level - tz;
}

__global__ void leaf_open_count(const u64* __restrict__ b, u64 leaves, int level, u32* __restrict__ cnt) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < leaves;
         i += (u64)gridDim.x * blockDim.x) {
        const int dl = leaf_depth(b[i + 1] - b[i], level);
        const int d0 = first_open_depth(b[i], level);
        cnt[i] = dl > d0 ? static_cast<u32>(dl - d0) : 0u;
    }
}

// exact-match lower_bound over the boundaries (the tiling guarantees the key is present)
__device__ __forceinline__ u64 find_boundary(const u64* __restrict__ b, u64 lo, u64 hi, u64 key) {
    while (lo < hi) {
        const u64 mid = (lo + hi) >> 1;
        if (b[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void leaf_link(const u64* __restrict__ b, const u32* __restrict__ off, u64 leaves,
                          int level, const u32* __restrict__ cnt, const u32* __restrict__ S,
                          lo_internal_node* __restrict__ nodes, u32* __restrict__ nchild) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < leaves;
         i += (u64)gridDim.x * blockDim.x) {
        const u32 c_i = cnt[i];
        if (!c_i) continue;
        const u64 s = b[i];
        const int d0 = first_open_depth(s, level);
        for (u32 j = 0; j < c_i; ++j) {
            const int d = d0 + static_cast<int>(j);
            const u64 blk = 1ull << (3 * (level - d)), sub = blk >> 3;
            const u64 e_leaf = find_boundary(b, i + 1, leaves + 1, s + blk);
            lo_internal_node nd;
            nd.prefix = s;
            nd.begin = off[i];
            nd.end = off[e_leaf];
            nd.depth = static_cast<u8>(d);
            u8 mask = 0;
            u64 jl = i;
            for (int c = 0; c < 8; ++c) {
                const u64 cs = s + c * sub;
                jl = find_boundary(b, jl, e_leaf, cs);
                const u64 ce = find_boundary(b, jl + 1, e_leaf + 1, cs + sub);
                i32 child;
                if (ce == jl + 1) {
                    child = ~static_cast<i32>(jl);  // the child block is one leaf
                } else {
                    const int dj0 = first_open_depth(b[jl], level);
                    child = static_cast<i32>(S[jl] + static_cast<u32>(d + 1 - dj0));
                }
                nd.children[c] = child;
                if (off[ce] != off[jl]) mask |= static_cast<u8>(1u << c);
            }
            nd.child_mask = mask;
            for (int q = 0; q < 6; ++q) nd.pad_[q] = 0;
            nodes[S[i] + j] = nd;
            nchild[S[i] + j] = __popc(mask);
        }
    }
}

// LinearOctree(LeafArray, ...) validation (linear_octree.cpp:88-103) and the device link of the
// internal nodes from the leaves alone (no cloud needed).
static LeafBuild link_leaf_array(lo_context* ctx, const u64* b_host, const u32* off_host, u64 count,
                                 const double disc_box[6], int level) {
    // Discretizer ctor (sfc.cpp:99-104)
    require(level >= 0 && level <= kMaxLevel, LO_INVALID_ARGUMENT, "level out of range");
    require(disc_box[0] <= disc_box[3] && disc_box[1] <= disc_box[4] && disc_box[2] <= disc_box[5],
            LO_INVALID_ARGUMENT, "inverted bounding box");
    const u64 full = 1ull << (3 * level);
    require(count >= 2 && b_host[0] == 0 && b_host[count - 1] == full && off_host[0] == 0,
            LO_INVALID_ARGUMENT, "linear octree: malformed leaf array");
    for (u64 i = 0; i + 1 < count; ++i) {
        const u64 span = b_host[i + 1] - b_host[i];
        const bool aligned_pow8 = b_host[i + 1] > b_host[i] && (span & (span - 1)) == 0 &&
                                  __builtin_ctzll(span) % 3 == 0 && b_host[i] % span == 0;
        if (!aligned_pow8 || off_host[i] > off_host[i + 1])
            throw Error(LO_INVALID_ARGUMENT, "linear octree: misaligned leaf span at " + std::to_string(i));
    }
    const u64 L = count - 1;
    LeafBuild lb;
    lb.leaves = L;
    lb.bounds = dalloc_t<u64>(ctx, count);
    lb.offsets = dalloc_t<u32>(ctx, count);
    LO_CUDA(cudaMemcpyAsync(lb.bounds, b_host, 8 * count, cudaMemcpyHostToDevice, ctx->stream));
    LO_CUDA(cudaMemcpyAsync(lb.offsets, off_host, 4 * count, cudaMemcpyHostToDevice, ctx->stream));
    u32* cnt = dalloc_t<u32>(ctx, L);
    u32* S = dalloc_t<u32>(ctx, L + 1);
    leaf_open_count<<<grid1(ctx, L), 256, 0, ctx->stream>>>(lb.bounds, L, level, cnt);
    LO_CHECK_LAUNCH();
    exclusive_scan_u32(ctx, cnt, S, L);
    const u32 I = read_scalar(ctx, S + L);
    lb.internal = I;
    lb.nodes = dalloc_t<lo_internal_node>(ctx, I);
    lb.nchild = dalloc_t<u32>(ctx, I + 1);
    if (I > 0) {
        leaf_link<<<grid1(ctx, L, 128), 128, 0, ctx->stream>>>(lb.bounds, lb.offsets, L, level, cnt, S,
                                                               lb.nodes, lb.nchild);
        LO_CHECK_LAUNCH();
    }
    dfree(ctx, cnt);
    dfree(ctx, S);
    return lb;
}

static void free_leaf_build(lo_context* ctx, LeafBuild& lb) {
    dfree(ctx, lb.bounds), dfree(ctx, lb.offsets), dfree(ctx, lb.nodes), dfree(ctx, lb.nchild);
    lb = LeafBuild{};
}

lo_octree* octree_from_leaves(lo_context* ctx, const lo_coded* coded, const u64* b_host,
                              const u32* off_host, u64 count, const double disc_box[6], int level,
                              int curve, u32 n_max) {
    require(coded != nullptr, LO_INVALID_ARGUMENT, "null coded cloud");
    stage_begin(ctx, "build");
    LeafBuild lb = link_leaf_array(ctx, b_host, off_host, count, disc_box, level);
    // the device tree searches this cloud: its leaves must index exactly its points
    if (!(off_host[count - 1] == coded->n && level == coded->level && curve == coded->curve)) {
        free_leaf_build(ctx, lb);
        throw Error(LO_INVALID_ARGUMENT, "linear octree: leaf array does not match the coded cloud");
    }
    lo_octree* t = finish_octree(ctx, coded, lb, n_max, level, curve, disc_box);
    stage_end(ctx);
    return t;
}

// Discretizer::octant_bounds (sfc.cpp:110-127) on the host: one padded box.
static void octant_bounds_host(const double box[6], int level, u32 hx, u32 hy, u32 hz, int depth, double out[6]) {
    require(level >= 0 && level <= kMaxLevel && depth >= 0 && depth <= level, LO_INVALID_ARGUMENT,
            "depth out of range");
    if (depth == 0) {
        std::memcpy(out, box, 6 * sizeof(double));
        return;
    }
    const double inv = std::ldexp(1.0, -depth);
    const u32 h[3] = {hx, hy, hz};
    for (int a = 0; a < 3; ++a) {
        const double side = (box[3 + a] - box[a]) * inv;
        const double lo = box[a] + h[a] * side;
        const double hi = lo + side;
        out[a] = dbl_from_order_key(dbl_order_key(lo) - 2);
        out[3 + a] = dbl_from_order_key(dbl_order_key(hi) + 2);
    }
}

}  // namespace lo

using namespace lo;

extern "C" {

int lo_build_leaves(lo_context* ctx, const uint64_t* codes_host, uint64_t n, uint32_t n_max,
                    int level, uint64_t* leaves, uint64_t* boundaries_host, uint32_t* offsets_host,
                    uint64_t cap) {
    return api_ctx(ctx, [&] {
        require(n_max >= 1, LO_INVALID_ARGUMENT, "build_leaves: n_max must be >= 1");
        require(n > 0, LO_INVALID_ARGUMENT, "build_leaves: empty code array");
        require(level >= 0 && level <= kMaxLevel, LO_INVALID_ARGUMENT, "level out of range");
        require(n <= 0xffffffffull, LO_INVALID_ARGUMENT, "build_leaves: too many codes");
        u64* codes = dalloc_t<u64>(ctx, n);
        LO_CUDA(cudaMemcpyAsync(codes, codes_host, 8 * n, cudaMemcpyHostToDevice, ctx->stream));
        try {
            validate_codes(ctx, codes, n, level);
        } catch (...) {
            dfree(ctx, codes);
            throw;
        }
        LeafBuild lb = build_tables(ctx, codes, n, n_max, level);
        *leaves = lb.leaves;
        if (boundaries_host && cap >= lb.leaves + 1) {
            LO_CUDA(cudaMemcpyAsync(boundaries_host, lb.bounds, 8 * (lb.leaves + 1),
                                    cudaMemcpyDeviceToHost, ctx->stream));
            LO_CUDA(cudaMemcpyAsync(offsets_host, lb.offsets, 4 * (lb.leaves + 1),
                                    cudaMemcpyDeviceToHost, ctx->stream));
        }
        dfree(ctx, codes);
        dfree(ctx, lb.bounds);
        dfree(ctx, lb.offsets);
        dfree(ctx, lb.nodes);
        dfree(ctx, lb.nchild);
        sync(ctx);
        require(boundaries_host == nullptr || cap >= lb.leaves + 1, LO_INVALID_ARGUMENT,
                "build_leaves: output capacity too small");
    });
}

int lo_octree_build(lo_context* ctx, const lo_coded* coded, uint32_t n_max, lo_octree** out) {
    return api_ctx(ctx, [&] { *out = octree_build(ctx, coded, n_max); });
}

int lo_octree_info_get(const lo_octree* t, lo_octree_info* out) {
    return api([&] {
        require(t != nullptr, LO_INVALID_ARGUMENT, "null octree");
        out->leaves = t->leaves;
        out->internal = t->internal;
        out->root = t->root;
        out->n_max = t->n_max;
        out->level = t->level;
        out->curve = t->curve;
        out->points = t->points;
        out->tnodes = t->tnodes;
    });
}

int lo_octree_download(lo_context* ctx, const lo_octree* t, uint64_t* boundaries_host,
                       uint32_t* offsets_host, lo_internal_node* nodes_host) {
    return api_ctx(ctx, [&] {
        if (boundaries_host)
            LO_CUDA(cudaMemcpyAsync(boundaries_host, t->bounds, 8 * (t->leaves + 1),
                                    cudaMemcpyDeviceToHost, ctx->stream));
        if (offsets_host)
            LO_CUDA(cudaMemcpyAsync(offsets_host, t->offsets, 4 * (t->leaves + 1),
                                    cudaMemcpyDeviceToHost, ctx->stream));
        if (nodes_host && t->internal)
            LO_CUDA(cudaMemcpyAsync(nodes_host, t->nodes, sizeof(lo_internal_node) * t->internal,
                                    cudaMemcpyDeviceToHost, ctx->stream));
        sync(ctx);
    });
}

int lo_link_leaves(lo_context* ctx, const uint64_t* boundaries_host, const uint32_t* offsets_host, uint64_t count,
                   const double disc_box[6], int level, uint64_t* internal, int32_t* root,
                   lo_internal_node* nodes_host, uint64_t cap) {
    return api_ctx(ctx, [&] {
        require(boundaries_host && offsets_host && disc_box && internal && root, LO_INVALID_ARGUMENT,
                "null argument");
        LeafBuild lb = link_leaf_array(ctx, boundaries_host, offsets_host, count, disc_box, level);
        *internal = lb.internal;
        *root = lb.internal > 0 ? 0 : ~0;
        if (nodes_host && lb.internal && cap >= lb.internal)
            LO_CUDA(cudaMemcpyAsync(nodes_host, lb.nodes, sizeof(lo_internal_node) * lb.internal,
                                    cudaMemcpyDeviceToHost, ctx->stream));
        sync(ctx);
        free_leaf_build(ctx, lb);
    });
}

int lo_octant_bounds(const double disc_box[6], int level, uint32_t hx, uint32_t hy, uint32_t hz, int depth,
                     double out[6]) {
    return api([&] {
        require(disc_box && out, LO_INVALID_ARGUMENT, "null argument");
        octant_bounds_host(disc_box, level, hx, hy, hz, depth, out);
    });
}

int lo_octree_node_bounds(lo_context* ctx, const lo_octree* t, const int32_t* refs_host,
                          uint64_t count, double* boxes_host) {
    return api_ctx(ctx, [&] {
        if (count == 0) return;
        for (u64 r = 0; r < count; ++r) {
            const i32 ref = refs_host[r];
            require(ref >= 0 ? static_cast<u64>(ref) < t->internal : static_cast<u64>(~ref) < t->leaves,
                    LO_INVALID_ARGUMENT, "node_bounds: NodeRef out of range");
        }
        i32* refs = dalloc_t<i32>(ctx, count);
        double* out = dalloc_t<double>(ctx, 6 * count);
        LO_CUDA(cudaMemcpyAsync(refs, refs_host, 4 * count, cudaMemcpyHostToDevice, ctx->stream));
        BoundsParams p{};
        std::memcpy(p.box, t->disc_box, sizeof p.box);
        p.level = t->level;
        std::memcpy(p.dec, curve_tables(t->curve).dec, sizeof p.dec);
        node_bounds_kernel<<<grid1(ctx, count), 256, 0, ctx->stream>>>(refs, count, t->nodes,
                                                                       t->bounds, p, out);
        LO_CHECK_LAUNCH();
        LO_CUDA(cudaMemcpyAsync(boxes_host, out, 48 * count, cudaMemcpyDeviceToHost, ctx->stream));
        dfree(ctx, refs);
        dfree(ctx, out);
        sync(ctx);
    });
}

int lo_octree_device_ptrs(const lo_octree* t, void** boundaries, void** offsets, void** nodes,
                          void** tnodes) {
    return api([&] {
        if (boundaries) *boundaries = t->bounds;
        if (offsets) *offsets = t->offsets;
        if (nodes) *nodes = t->nodes;
        if (tnodes) *tnodes = t->tn;
    });
}

int lo_octree_create_empty(lo_context* ctx, const lo_coded* coded, const lo_octree_info* info,
                           lo_octree** out) {
    return api_ctx(ctx, [&] {
        require(coded && info && info->points == coded->n, LO_INVALID_ARGUMENT,
                "octree header does not match the coded cloud");
        auto* t = new lo_octree;
        t->ctx = ctx;
        t->coded = coded;
        t->points = info->points;
        t->leaves = info->leaves;
        t->internal = info->internal;
        t->tnodes = info->tnodes;
        t->root = info->root;
        t->n_max = info->n_max;
        t->level = info->level;
        t->curve = info->curve;
        std::memcpy(t->disc_box, coded->disc_box, sizeof t->disc_box);
        try {
            t->bounds = dalloc_t<u64>(ctx, t->leaves + 1);
            t->offsets = dalloc_t<u32>(ctx, t->leaves + 1);
            t->nodes = dalloc_t<lo_internal_node>(ctx, t->internal);
            t->tn = dalloc_t<TNode>(ctx, t->tnodes);
            sync(ctx);
        } catch (...) {
            dfree(ctx, t->bounds), dfree(ctx, t->offsets), dfree(ctx, t->nodes), dfree(ctx, t->tn);
            delete t;
            throw;
        }
        *out = t;
    });
}

int lo_octree_destroy(lo_octree* t) {
    if (!t) return LO_OK;
    return api_ctx(t->ctx, [&] {
        lo_context* ctx = t->ctx;
        if (t->reader) {  // a broadcast / peer copy may still read the buffers: free behind it
            LO_CUDA(cudaStreamWaitEvent(ctx->stream, t->reader, 0));
            cudaEventDestroy(t->reader);
        }
        dfree(ctx, t->bounds);
        dfree(ctx, t->offsets);
        dfree(ctx, t->nodes);
        dfree(ctx, t->tn);
        dfree(ctx, t->tf);
        dfree(ctx, t->rb);
        dfree(ctx, t->rbf);
        delete t;
    });
}

}  // extern "C"
