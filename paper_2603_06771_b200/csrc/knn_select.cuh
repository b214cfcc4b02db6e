// knn_select.cuh -- kNN by bounded candidate collection and warp-wide selection (k <= 64), included
// by knn.cu.  Replaces the per-lane heaps of knn_float.cuh for Full / range / curve-sorted centre
// batches; the result is the same (index, dist_sq) rows as knn_lin_oct (search.cpp:190-252).
//
// Three kernels per chunk of queries:
//   K7a knn_bound_kernel   (warp per query)  w = an upper bound of the k-th smallest FP64 dist_sq:
//       the k-th smallest among the W points around the query along the curve (its own cloud
//       index +- W/2), found by a radix select over the top 13 bits of the FP32 round-up of their
//       FP64 distances (so w >= the window's k-th smallest >= the true k-th smallest).  The FP32
//       filter threshold T = knn_threshold(w) then admits every point with FP64 dist_sq <= w.
//   K7b knn_collect_kernel (lane = query, warp = 32 consecutive queries)  the octree walk of
//       knn_float_kernel with the per-query threshold T fixed: every point whose FP32 filter
//       distance is <= T is appended to the query's candidate list (capacity `cap`), each leaf
//       is visited at most once per tile, so a list has no duplicates.  This set contains the k
//       nearest points (every point with dist_sq <= w passes), typically 1.4-2x k of them.
//   K7c knn_select_kernel  (warp per query)  the candidates' FP64 distances (reference
//       expression), a warp-wide bitonic sort of the 64-bit keys (FP32 round-up of dist_sq << 32 |
//       index), then the first k written with coalesced stores.  The round-up is monotone, so
//       keys with different high words order exactly; runs of equal high words that reach into
//       the first k are re-sorted by the exact (dist_sq, index) (rare; one lane).
// A query whose list overflows `cap` (a sparse point, a curve jump) is recomputed by the heap
// kernel (`fallback`) and its row scattered into place.
#pragma once

namespace lo {

constexpr int kKsWarps = 4;

__device__ __forceinline__ u64 ks_anchor(const Queries& q, i64 seed_base, u64 qi) {
    return seed_base >= 0 ? static_cast<u64>(seed_base) + qi : static_cast<u64>(q.idx[qi]);
}

template <int M>
__global__ void __launch_bounds__(128) knn_bound_kernel(const double* __restrict__ px, const double* __restrict__ py,
                                                        const double* __restrict__ pz, u64 n, Queries q, i64 seed_base,
                                                        u64 q0, u64 mc, u32 k, float E, float* __restrict__ t_out) {
    constexpr u32 W = 32 * M;
    const int lane = threadIdx.x & 31;
    const u64 nw = (static_cast<u64>(gridDim.x) * blockDim.x) >> 5;
    for (u64 i = (static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < mc; i += nw) {
        const u64 qi = q0 + i;
        double cx, cy, cz;
        load_query(q, qi, cx, cy, cz);
        const i64 a = static_cast<i64>(ks_anchor(q, seed_base, qi));
        i64 lo = a - static_cast<i64>(W / 2);
        if (lo + static_cast<i64>(W) > static_cast<i64>(n)) lo = static_cast<i64>(n) - static_cast<i64>(W);
        if (lo < 0) lo = 0;
        u32 key[M];
#pragma unroll
        for (int j = 0; j < M; ++j) {
            const u64 g = static_cast<u64>(lo) + 32 * j + lane;
            key[j] = g < n ? __float_as_uint(__double2float_ru(
                                 point_dist_sq(__ldg(px + g), __ldg(py + g), __ldg(pz + g), cx, cy, cz)))
                           : 0x7f800000u;
        }
        // radix select of the k-th smallest key on bits 30..18 (positive floats order as u32)
        u32 prefix = 0, kk = k;
#pragma unroll 1
        for (int b = 30; b >= 18; --b) {
            const u32 want = prefix >> b;
            u32 cnt = 0;
#pragma unroll
            for (int j = 0; j < M; ++j) cnt += (key[j] >> b) == want ? 1u : 0u;
            cnt = __reduce_add_sync(~0u, cnt);
            if (cnt < kk) {
                kk -= cnt;
                prefix |= 1u << b;
            }
        }
        // every key with these top bits is <= prefix | 0x3ffff: at least k window points have
        // FP64 dist_sq <= w
        const float w = __uint_as_float(prefix | 0x3ffffu);
        if (lane == 0) t_out[i] = knn_threshold(static_cast<double>(w), E);
    }
}

// Per-warp shared layout of knn_collect_kernel (bytes): stack | tq | qf | pa | pb | pidx | sidx
constexpr size_t kKcOffStack = 0;
constexpr size_t kKcOffTq = kKcOffStack + 4 * kStackCap;
constexpr size_t kKcOffQf = kKcOffTq + 4 * 32;
constexpr size_t kKcOffPa = kKcOffQf + 16 * 32;
constexpr size_t kKcOffPb = kKcOffPa + 16 * 16;
constexpr size_t kKcOffPidx = kKcOffPb + 8 * 16;
constexpr size_t kKcOffSidx = kKcOffPidx + 4 * 32;
constexpr size_t kKcFixed = kKcOffSidx + 4 * 32;

__global__ void __launch_bounds__(32 * kKsWarps) knn_collect_kernel(
    const TNodeF* __restrict__ tf, const float4* __restrict__ pf, Queries q, u64 q0, u64 mc,
    const float* __restrict__ tq_in, u32 cap, u32* __restrict__ lists, u32* __restrict__ counts,
    u64* tile_counter) {
    __shared__ __align__(16) unsigned char smem[kKsWarps * kKcFixed];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned char* mine = smem + w * kKcFixed;
    u32* stack = reinterpret_cast<u32*>(mine + kKcOffStack);
    float* tq = reinterpret_cast<float*>(mine + kKcOffTq);
    float4* qfs = reinterpret_cast<float4*>(mine + kKcOffQf);
    float* pa = reinterpret_cast<float*>(mine + kKcOffPa);
    float* pb = reinterpret_cast<float*>(mine + kKcOffPb);
    u32* pidx = reinterpret_cast<u32*>(mine + kKcOffPidx);
    u32* sidx = reinterpret_cast<u32*>(mine + kKcOffSidx);
    const u64 ntiles = (mc + 31) / 32;
    const int cl = lane & 7, grp = lane >> 3;
    for (;;) {
        u64 tile = 0;
        if (lane == 0) tile = atomicAdd(reinterpret_cast<unsigned long long*>(tile_counter), 1ull);
        tile = __shfl_sync(~0u, tile, 0);
        if (tile >= ntiles) break;
        const u64 i = tile * 32 + lane;
        const bool active = i < mc;
        float4 qf = make_float4(INFINITY, INFINITY, INFINITY, 0.f);
        float T = -INFINITY;  // inactive lanes want nothing
        if (active) {
            qf = load_query_f(q, q0 + i);
            T = tq_in[i];
        }
        const u64 QX = pack2(qf.x, qf.x), QY = pack2(qf.y, qf.y), QZ = pack2(qf.z, qf.z);
        u32* list = lists + (active ? i : 0) * cap;
        u32 cnt = 0;
        __syncwarp();
        qfs[lane] = qf;
        tq[lane] = T;
        u32 kfill = 0;
        bool kwant = false;
        // test the kfill gathered candidates against this lane's query, append the ones under T
        auto flush = [&]() {
            __syncwarp();
            if (static_cast<u32>(lane) < kfill) {
                const u32 g = sidx[lane];
                const float4 p = __ldg(pf + g);
                const int pp = lane >> 1, h = lane & 1;
                pa[4 * pp + h] = p.x;
                pa[4 * pp + 2 + h] = p.y;
                pb[2 * pp + h] = p.z;
                pidx[lane] = g;
            }
            __syncwarp();
            if (kwant) {
                const u32 npairs = (kfill + 1) >> 1;
                for (u32 pp = 0; pp < npairs; ++pp) {
                    const float4 A = reinterpret_cast<const float4*>(pa)[pp];
                    const float2 B = reinterpret_cast<const float2*>(pb)[pp];
                    const u64 dx = fsub2(pack2(A.x, A.y), QX);
                    const u64 dy = fsub2(pack2(A.z, A.w), QY);
                    const u64 dz = fsub2(pack2(B.x, B.y), QZ);
                    u64 d2 = fmul2(dx, dx);
                    d2 = ffma2(dy, dy, d2);
                    d2 = ffma2(dz, dz, d2);
                    float v0, v1;
                    unpack2(d2, v0, v1);
                    if (v0 <= T) {
                        if (cnt < cap) list[cnt] = pidx[2 * pp];
                        ++cnt;
                    }
                    if (2 * pp + 1 < kfill && v1 <= T) {
                        if (cnt < cap) list[cnt] = pidx[2 * pp + 1];
                        ++cnt;
                    }
                }
            }
            kfill = 0;
            kwant = false;
        };
        int sp = 1;
        if (lane == 0) stack[0] = 0;
        __syncwarp();
        while (sp > 0) {
            __syncwarp();
            const u32 t = stack[--sp];
            const NodeF nd = load_node_f(tf, t);
            if (nd.nchild != 0) {
                bool keep = false;
                if (cl < static_cast<int>(nd.nchild)) {
                    const NodeF ch = load_node_f(tf, nd.child0 + cl);
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const float4 qq = qfs[8 * grp + j];
                        const float nx = fmaxf(fmaxf(ch.lo[0] - qq.x, qq.x - ch.hi[0]), 0.f);
                        const float ny = fmaxf(fmaxf(ch.lo[1] - qq.y, qq.y - ch.hi[1]), 0.f);
                        const float nz = fmaxf(fmaxf(ch.lo[2] - qq.z, qq.z - ch.hi[2]), 0.f);
                        keep |= fmaf(nz, nz, fmaf(ny, ny, nx * nx)) <= tq[8 * grp + j];
                    }
                }
                u32 s = __ballot_sync(~0u, keep);
                s = (s | (s >> 8) | (s >> 16) | (s >> 24)) & 0xffu;
                const int kk = __popc(s);
                __syncwarp();
                if (lane < 8 && ((s >> lane) & 1u))
                    stack[sp + kk - 1 - __popc(s & ((1u << lane) - 1u))] = nd.child0 + lane;
                sp += kk;
                continue;
            }
            bool want = false;
            if (active) {
                const float nx = fmaxf(fmaxf(nd.lo[0] - qf.x, qf.x - nd.hi[0]), 0.f);
                const float ny = fmaxf(fmaxf(nd.lo[1] - qf.y, qf.y - nd.hi[1]), 0.f);
                const float nz = fmaxf(fmaxf(nd.lo[2] - qf.z, qf.z - nd.hi[2]), 0.f);
                want = fmaf(nz, nz, fmaf(ny, ny, nx * nx)) <= T;
            }
            if (!__any_sync(~0u, want)) continue;
            for (u32 b = nd.begin; b < nd.end;) {
                const u32 take = min(32u - kfill, nd.end - b);
                __syncwarp();
                if (static_cast<u32>(lane) < take) sidx[kfill + lane] = b + lane;
                kfill += take;
                kwant |= want;
                b += take;
                if (kfill == 32) flush();
            }
        }
        if (kfill) flush();
        if (active) counts[i] = cnt;
    }
}

__device__ __forceinline__ u64 ks_min(u64 a, u64 b) { return a < b ? a : b; }
__device__ __forceinline__ u64 ks_max(u64 a, u64 b) { return a < b ? b : a; }

// Ascending bitonic sort of 32 * M keys held as element e = 32 * j + lane in v[j].
template <int M>
__device__ __forceinline__ void ks_bitonic(u64 (&v)[M], int lane) {
    constexpr int S = 32 * M;
#pragma unroll
    for (int s = 2; s <= S; s <<= 1) {
#pragma unroll
        for (int d = s >> 1; d > 0; d >>= 1) {
            if (d >= 32) {
                const int dj = d >> 5;
#pragma unroll
                for (int j = 0; j < M; ++j) {
                    if ((j & dj) == 0) {
                        const bool asc = ((32 * j) & s) == 0;
                        const u64 a = v[j], b = v[j | dj];
                        const bool sw = asc ? (b < a) : (a < b);
                        v[j] = sw ? b : a;
                        v[j | dj] = sw ? a : b;
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < M; ++j) {
                    const u64 p = __shfl_xor_sync(~0u, v[j], d);
                    const bool asc = ((32 * j + lane) & s) == 0;
                    const bool lower = (lane & d) == 0;
                    v[j] = (lower == asc) ? ks_min(v[j], p) : ks_max(v[j], p);
                }
            }
        }
    }
}

// One query's row from its c (k <= c <= 32 * M) candidates.
template <int M>
__device__ __forceinline__ void ks_row(const u32* __restrict__ list, u32 c, u32 k, int lane, double cx, double cy,
                                       double cz, const double* __restrict__ px, const double* __restrict__ py,
                                       const double* __restrict__ pz, u64* sm, u32* __restrict__ oi,
                                       double* __restrict__ od) {
    u64 v[M];
#pragma unroll
    for (int j = 0; j < M; ++j) {
        const u32 e = 32 * j + lane;
        v[j] = ~0ull;
        if (e < c) {
            const u32 g = list[e];
            const double d = point_dist_sq(__ldg(px + g), __ldg(py + g), __ldg(pz + g), cx, cy, cz);
            v[j] = static_cast<u64>(__float_as_uint(__double2float_ru(d))) << 32 | g;
        }
    }
    ks_bitonic<M>(v, lane);
#pragma unroll
    for (int j = 0; j < M; ++j) sm[32 * j + lane] = v[j];
    __syncwarp();
    // equal high words (FP32 keys) that reach into the first k: exact order decides
    bool tie = false;
    for (u32 e = lane + 1; e <= k && e < c; e += 32) tie |= (sm[e] >> 32) == (sm[e - 1] >> 32);
    if (__any_sync(~0u, tie)) {
        if (lane == 0) {
            u32 a = 0;
            while (a < k) {
                u32 b = a + 1;
                while (b < c && (sm[b] >> 32) == (sm[a] >> 32)) ++b;
                for (u32 x = a + 1; x < b; ++x) {  // insertion sort by (dist_sq, index)
                    const u64 kx = sm[x];
                    const u32 gx = static_cast<u32>(kx);
                    const double dx = point_dist_sq(px[gx], py[gx], pz[gx], cx, cy, cz);
                    u32 y = x;
                    while (y > a) {
                        const u32 gy = static_cast<u32>(sm[y - 1]);
                        const double dy = point_dist_sq(px[gy], py[gy], pz[gy], cx, cy, cz);
                        if (dy < dx || (dy == dx && gy < gx)) break;
                        sm[y] = sm[y - 1];
                        --y;
                    }
                    sm[y] = kx;
                }
                a = b;
            }
        }
        __syncwarp();
    }
    for (u32 e = lane; e < k; e += 32) {
        const u32 g = static_cast<u32>(sm[e]);
        oi[e] = g;
        od[e] = point_dist_sq(__ldg(px + g), __ldg(py + g), __ldg(pz + g), cx, cy, cz);
    }
    __syncwarp();
}

__global__ void __launch_bounds__(32 * kKsWarps) knn_select_kernel(
    const double* __restrict__ px, const double* __restrict__ py, const double* __restrict__ pz, Queries q,
    i64 seed_base, u64 q0, u64 mc, u32 k, u32 cap, const u32* __restrict__ lists, const u32* __restrict__ counts,
    u32* __restrict__ out_idx, double* __restrict__ out_dist, u32* __restrict__ ovf_anchor,
    u32* __restrict__ ovf_row, u32* ovf_n) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    u64* sm = reinterpret_cast<u64*>(smem) + static_cast<u64>(w) * cap;
    const u64 nw = (static_cast<u64>(gridDim.x) * blockDim.x) >> 5;
    for (u64 i = (static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < mc; i += nw) {
        const u64 qi = q0 + i;
        const u32 c = counts[i];
        if (c > cap || c < k) {  // overflow (c < k cannot happen: the window's k points pass)
            if (lane == 0) {
                const u32 s = atomicAdd(ovf_n, 1u);
                ovf_anchor[s] = static_cast<u32>(ks_anchor(q, seed_base, qi));
                ovf_row[s] = static_cast<u32>(qi);
            }
            continue;
        }
        double cx, cy, cz;
        load_query(q, qi, cx, cy, cz);
        const u32* list = lists + i * cap;
        u32* oi = out_idx + qi * k;
        double* od = out_dist + qi * k;
        const u32 m = (c + 31) / 32;
        if (m <= 1) ks_row<1>(list, c, k, lane, cx, cy, cz, px, py, pz, sm, oi, od);
        else if (m <= 2) ks_row<2>(list, c, k, lane, cx, cy, cz, px, py, pz, sm, oi, od);
        else if (m <= 4) ks_row<4>(list, c, k, lane, cx, cy, cz, px, py, pz, sm, oi, od);
        else if (m <= 8) ks_row<8>(list, c, k, lane, cx, cy, cz, px, py, pz, sm, oi, od);
        else ks_row<16>(list, c, k, lane, cx, cy, cz, px, py, pz, sm, oi, od);
    }
}

// Rows of the fallback batch (heap kernel) into their places.
__global__ void knn_scatter_rows(const u32* __restrict__ ti, const double* __restrict__ td,
                                 const u32* __restrict__ rows, u32 n, u32 k, u32* __restrict__ out_idx,
                                 double* __restrict__ out_dist) {
    const u64 total = static_cast<u64>(n) * k;
    for (u64 e = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<u64>(gridDim.x) * blockDim.x) {
        const u64 r = e / k, j = e - r * k;
        const u64 o = static_cast<u64>(rows[r]) * k + j;
        out_idx[o] = ti[e];
        out_dist[o] = td[e];
    }
}

inline u32 ks_env(const char* name, u32 dflt) {
    const char* e = std::getenv(name);
    return e && *e ? static_cast<u32>(std::strtoul(e, nullptr, 10)) : dflt;
}
inline u32 ks_pow2(u32 v) {
    u32 p = 1;
    while (p < v) p <<= 1;
    return p;
}

// Runs the three kernels over chunks of the batch; `fallback(queries, seed_base, idx, dist)` runs
// the heap kernel for the overflowed queries.
template <class Fallback>
void knn_select_run(lo_context* ctx, const lo_octree* t, const lo_coded* c, const Queries& q, u32 k, i64 seed_base,
                    float E, u32* out_idx, double* out_dist, Fallback&& fallback) {
    // window of the bound: LO_KNN_WIN x k points (default 4), in whole warps
    const u32 mb = std::min<u32>(16, ks_pow2(std::max<u32>(1, (ks_env("LO_KNN_WIN", 4) * k + 31) / 32)));
    // candidate list capacity: LO_KNN_CAP x k (default 8), a power of two in [32, 512]
    const u32 cap = std::min<u32>(512, std::max<u32>(32, ks_pow2(ks_env("LO_KNN_CAP", 8) * k)));
    const u64 budget = static_cast<u64>(ks_env("LO_KNN_LIST_MB", 8192)) << 20;
    u64 chunk = std::max<u64>(32 * 1024, budget / (4ull * cap));
    chunk = std::min<u64>(chunk, q.m);
    float* tq = nullptr;
    u32 *counts = nullptr, *lists = nullptr, *ovf = nullptr, *ovf_n = nullptr;
    u64* counter = nullptr;
    u32* ti = nullptr;
    double* td = nullptr;
    try {
        tq = dalloc_t<float>(ctx, chunk);
        counts = dalloc_t<u32>(ctx, chunk);
        lists = dalloc_t<u32>(ctx, chunk * cap);
        ovf = dalloc_t<u32>(ctx, 2 * chunk);
        ovf_n = dalloc_t<u32>(ctx, 1);
        counter = dalloc_t<u64>(ctx, 1);
        const int sms = ctx->sm_count;
        const int bblocks = static_cast<int>(std::min<u64>((chunk + kKsWarps - 1) / kKsWarps, static_cast<u64>(sms) * 16));
        const size_t sel_smem = static_cast<size_t>(kKsWarps) * cap * 8;
        for (u64 q0 = 0; q0 < q.m; q0 += chunk) {
            const u64 mc = std::min<u64>(chunk, q.m - q0);
            switch (mb) {
                case 1: knn_bound_kernel<1><<<bblocks, 128, 0, ctx->stream>>>(c->x, c->y, c->z, c->n, q, seed_base, q0, mc, k, E, tq); break;
                case 2: knn_bound_kernel<2><<<bblocks, 128, 0, ctx->stream>>>(c->x, c->y, c->z, c->n, q, seed_base, q0, mc, k, E, tq); break;
                case 4: knn_bound_kernel<4><<<bblocks, 128, 0, ctx->stream>>>(c->x, c->y, c->z, c->n, q, seed_base, q0, mc, k, E, tq); break;
                case 8: knn_bound_kernel<8><<<bblocks, 128, 0, ctx->stream>>>(c->x, c->y, c->z, c->n, q, seed_base, q0, mc, k, E, tq); break;
                default: knn_bound_kernel<16><<<bblocks, 128, 0, ctx->stream>>>(c->x, c->y, c->z, c->n, q, seed_base, q0, mc, k, E, tq); break;
            }
            LO_CHECK_LAUNCH();
            LO_CUDA(cudaMemsetAsync(counter, 0, 8, ctx->stream));
            const u64 tiles = (mc + 31) / 32;
            const int cblocks = static_cast<int>(std::max<u64>(1, std::min<u64>((tiles + kKsWarps - 1) / kKsWarps,
                                                                               static_cast<u64>(sms) * 16)));
            knn_collect_kernel<<<cblocks, 32 * kKsWarps, 0, ctx->stream>>>(t->tf, c->pf, q, q0, mc, tq, cap, lists,
                                                                           counts, counter);
            LO_CHECK_LAUNCH();
            LO_CUDA(cudaMemsetAsync(ovf_n, 0, 4, ctx->stream));
            knn_select_kernel<<<bblocks, 32 * kKsWarps, sel_smem, ctx->stream>>>(
                c->x, c->y, c->z, q, seed_base, q0, mc, k, cap, lists, counts, out_idx, out_dist, ovf, ovf + chunk,
                ovf_n);
            LO_CHECK_LAUNCH();
            const u32 n_ovf = read_scalar(ctx, ovf_n);
            static const bool debug = std::getenv("LO_DEBUG") != nullptr;
            if (debug)
                std::fprintf(stderr, "[lo] knn select: chunk %llu+%llu, cap %u, window %u: %u overflowed\n",
                             static_cast<unsigned long long>(q0), static_cast<unsigned long long>(mc), cap, 32 * mb,
                             n_ovf);
            if (n_ovf) {
                ti = dalloc_t<u32>(ctx, static_cast<u64>(n_ovf) * k);
                td = dalloc_t<double>(ctx, static_cast<u64>(n_ovf) * k);
                const Queries q2{c->x, c->y, c->z, ovf, n_ovf, c->pf, c->bmax};
                fallback(q2, kSeedSortedIdx, ti, td);
                knn_scatter_rows<<<std::max(1, std::min(sms * 8, ceil_div(static_cast<u64>(n_ovf) * k, 256))), 256, 0,
                                   ctx->stream>>>(ti, td, ovf + chunk, n_ovf, k, out_idx, out_dist);
                LO_CHECK_LAUNCH();
                dfree(ctx, ti), ti = nullptr;
                dfree(ctx, td), td = nullptr;
            }
        }
    } catch (...) {
        dfree(ctx, tq), dfree(ctx, counts), dfree(ctx, lists), dfree(ctx, ovf), dfree(ctx, ovf_n), dfree(ctx, counter);
        dfree(ctx, ti), dfree(ctx, td);
        throw;
    }
    dfree(ctx, tq), dfree(ctx, counts), dfree(ctx, lists), dfree(ctx, ovf), dfree(ctx, ovf_n), dfree(ctx, counter);
}

}  // namespace lo
