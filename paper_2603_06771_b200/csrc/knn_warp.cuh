// knn_warp.cuh -- warp-cooperative exact kNN for k <= 64 (K7 v2), included by knn.cu.
//
// knn_lin_oct (search.cpp:190-252) returns the first k points under (dist_sq, index), dist_sq the
// FP64 point_dist_sq (search.cpp:180-185).  The first kernel (knn_float.cuh) gave every lane its
// own query and a per-lane heap in shared memory: the sifts diverge (17 of 32 lanes active at
// k = 64) and occupancy is bound by 32 heaps per warp.  Here the warp works like the radius count
// (radius_pt.cuh): one warp owns 32 consecutive queries and walks the octree once for all of
// them, leaf points are gathered into a 32-slot buffer, and every buffer is tested lane =
// candidate against one query after the other:
//   * FP32 distances of the 32 candidates to query L (tile-local coordinates, see
//     radius_pt.cuh::tile_test), one ballot against L's threshold T_L;
//   * the few that pass get their exact FP64 dist_sq (the reference expression, no FMA) and are
//     inserted one by one into L's sorted top-k list, which is spread over the lanes (entry e in
//     lane e % 32, register e / 32): rank = popcount of a ballot, shift = one shuffle -- no
//     divergence, every lane busy;
//   * once L's list is full, T_L = worst + M(worst) (knn_float.cuh::knn_threshold): candidates
//     above it provably cannot enter.
// Node pruning uses a second threshold per query for the cloud-origin FP32 node boxes.  The
// lists are sorted as they grow, so the output needs no final sort.  Ties at the k-th distance
// resolve by index exactly as the reference's (dist_sq, index) order.
#pragma once

#include "knn_float.cuh"

namespace lo {

constexpr int kKwWarps = 4;

struct KwShared {
    u32 stack[kStackCap];
    u32 sidx[32];           // gathered leaf point indices (walk buffer)
    float4 qf[32];          // queries, FP32 relative to the cloud origin (node tests)
    float qx[32], qy[32], qz[32];  // queries, FP32 relative to the tile origin (point tests)
    double qd[32][3];       // queries, FP64
    float tg[32];           // node threshold per query (+inf until its list is full)
    float tl[32];           // point threshold per query
    u32 ls[32];             // list sizes
    u32 sklo[32], skhi[32]; // per query: seed window [lo, hi) already offered
};

// T(w) for the tile-local point test: the coordinates' error is 2^-24 |p - o_t| <= 2^-24 (ext +
// |p - q|) for the candidates that matter (|p - q| <= sqrt(w)); E = 2^-23 (ext + 2 sqrt(w)) bounds
// it with a factor-2 slack, then knn_threshold's M(w) as for the cloud origin.
__device__ __forceinline__ float kw_threshold_local(double w, float ext) {
    const float u = 1.1920928955078125e-07f;
    const float sw = __fsqrt_ru(__double2float_ru(w));
    const float E = __fmul_ru(u, __fmaf_ru(2.0f, sw, ext));
    return knn_threshold(w, E);
}

__device__ __forceinline__ bool kw_less(double ad, u32 ai, double bd, u32 bi) {
    return ad < bd || (ad == bd && ai < bi);
}

// Offers the lane's candidate (g, FP32 tile coordinates P, FP64 coordinates pd) to every query of
// qmask, one query after the other.  `skip`: drop candidates inside the query's seed window.
template <int R>
__device__ __forceinline__ void kw_buffer(KwShared& S, double* __restrict__ LD, u32* __restrict__ LI, u32 k,
                                          bool valid, u32 g, const float4& P, const double (&pd)[3], u32 qmask,
                                          bool skip, float ext, float E, int lane) {
    while (qmask) {
        const int L = __ffs(qmask) - 1;
        qmask &= qmask - 1;
        const float dx = P.x - S.qx[L], dy = P.y - S.qy[L], dz = P.z - S.qz[L];
        const float v = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
        bool ok = valid && v <= S.tl[L];
        if (skip) ok = ok && (g < S.sklo[L] || g >= S.skhi[L]);
        u32 pass = __ballot_sync(~0u, ok);
        if (!pass) continue;
        // exact FP64 dist_sq of the passing candidates (reference expression, search.cpp:180-185)
        const double d = ok ? point_dist_sq(pd[0], pd[1], pd[2], S.qd[L][0], S.qd[L][1], S.qd[L][2]) : 0.0;
        u32 size = S.ls[L];
        double* ld = LD + static_cast<u64>(L) * k;
        u32* li = LI + static_cast<u64>(L) * k;
        double ed[R];
        u32 ei[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const u32 p = lane + 32 * r;
            ed[r] = p < size ? ld[p] : INFINITY;
            ei[r] = p < size ? li[p] : ~0u;
        }
        const int wl = (k - 1) & 31, wr = (k - 1) >> 5;
        while (pass) {
            const int j = __ffs(pass) - 1;
            pass &= pass - 1;
            const double dn = __shfl_sync(~0u, d, j);
            const u32 in = __shfl_sync(~0u, g, j);
            if (size == k) {  // full: it must beat the current k-th (dist_sq, index)
                double wd = ed[0];
                u32 wi = ei[0];
#pragma unroll
                for (int r = 1; r < R; ++r)
                    if (wr == r) wd = ed[r], wi = ei[r];
                wd = __shfl_sync(~0u, wd, wl);
                wi = __shfl_sync(~0u, wi, wl);
                if (!kw_less(dn, in, wd, wi)) continue;
            }
            u32 pos = 0;
#pragma unroll
            for (int r = 0; r < R; ++r)
                pos += __popc(__ballot_sync(~0u, lane + 32 * r < static_cast<int>(size) && kw_less(ed[r], ei[r], dn, in)));
            // shift the tail one slot up (entry e -> e + 1) and drop the new entry at pos
            double carry_d = 0.0;
            u32 carry_i = 0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const double up_d = __shfl_up_sync(~0u, ed[r], 1);
                const u32 up_i = __shfl_up_sync(~0u, ei[r], 1);
                const double top_d = __shfl_sync(~0u, ed[r], 31);
                const u32 top_i = __shfl_sync(~0u, ei[r], 31);
                const u32 p = lane + 32 * r;
                const double prev_d = lane == 0 ? carry_d : up_d;
                const u32 prev_i = lane == 0 ? carry_i : up_i;
                if (p == pos) {
                    ed[r] = dn;
                    ei[r] = in;
                } else if (p > pos) {
                    ed[r] = prev_d;
                    ei[r] = prev_i;
                }
                carry_d = top_d;
                carry_i = top_i;
            }
            if (size < k) ++size;
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const u32 p = lane + 32 * r;
            if (p < size) {
                ld[p] = ed[r];
                li[p] = ei[r];
            }
        }
        if (size == k) {
            double wd = ed[0];
#pragma unroll
            for (int r = 1; r < R; ++r)
                if (wr == r) wd = ed[r];
            wd = __shfl_sync(~0u, wd, wl);
            if (lane == 0) {
                S.tl[L] = kw_threshold_local(wd, ext);
                S.tg[L] = knn_threshold(wd, E);
            }
        }
        if (lane == 0) S.ls[L] = size;
        __syncwarp();
    }
}

template <int R>
__global__ void __launch_bounds__(32 * kKwWarps) knn_warp_kernel(
    const TNodeF* __restrict__ tf, const double* __restrict__ px, const double* __restrict__ py,
    const double* __restrict__ pz, u64 npoints, Queries q, i64 seed_base, u32 seed_half, float E, u32 k,
    u32* __restrict__ out_idx, double* __restrict__ out_dist, u64* tile_counter) {
    extern __shared__ __align__(16) unsigned char kw_smem[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const size_t per_warp = (sizeof(KwShared) + 15) / 16 * 16 + static_cast<size_t>(32) * k * 12;
    unsigned char* mine = kw_smem + w * per_warp;
    KwShared& S = *reinterpret_cast<KwShared*>(mine);
    double* LD = reinterpret_cast<double*>(mine + (sizeof(KwShared) + 15) / 16 * 16);  // [32][k]
    u32* LI = reinterpret_cast<u32*>(LD + 32 * k);                                     // [32][k]
    const u64 ntiles = (q.m + 31) / 32;
    const int cl = lane & 7, grp = lane >> 3;
    for (;;) {
        u64 tile = 0;
        if (lane == 0) tile = atomicAdd(reinterpret_cast<unsigned long long*>(tile_counter), 1ull);
        tile = __shfl_sync(~0u, tile, 0);
        if (tile >= ntiles) break;
        const u64 qi = tile * 32 + lane;
        const bool active = qi < q.m;
        double cx = 0.0, cy = 0.0, cz = 0.0;
        float4 qf = make_float4(INFINITY, INFINITY, INFINITY, 0.f);
        if (active) {
            load_query(q, qi, cx, cy, cz);
            qf = load_query_f(q, qi);
        }
        const double ox = __shfl_sync(~0u, cx, 0), oy = __shfl_sync(~0u, cy, 0), oz = __shfl_sync(~0u, cz, 0);
        float ext = 0.f;
        __syncwarp();
        S.qf[lane] = qf;
        if (active) {
            S.qx[lane] = __double2float_rn(cx - ox);
            S.qy[lane] = __double2float_rn(cy - oy);
            S.qz[lane] = __double2float_rn(cz - oz);
            ext = __double2float_ru(fmax(fmax(fabs(cx - ox), fabs(cy - oy)), fabs(cz - oz)));
        } else {
            S.qx[lane] = S.qy[lane] = S.qz[lane] = INFINITY;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ext = fmaxf(ext, __shfl_xor_sync(~0u, ext, o));
        S.qd[lane][0] = cx;
        S.qd[lane][1] = cy;
        S.qd[lane][2] = cz;
        S.tg[lane] = active ? INFINITY : -INFINITY;  // inactive lanes want nothing
        S.tl[lane] = active ? INFINITY : -INFINITY;
        S.ls[lane] = 0;
        S.sklo[lane] = S.skhi[lane] = 0;
        const u32 act = __ballot_sync(~0u, active);
        __syncwarp();
        // a candidate in the lanes: FP32 tile coordinates + FP64 coordinates
        auto load_cand = [&](bool valid, u32 g, float4& P, double (&pd)[3]) {
            if (valid) {
                pd[0] = __ldg(px + g), pd[1] = __ldg(py + g), pd[2] = __ldg(pz + g);
                P = make_float4(__double2float_rn(pd[0] - ox), __double2float_rn(pd[1] - oy),
                                __double2float_rn(pd[2] - oz), 0.f);
            } else {
                pd[0] = pd[1] = pd[2] = 0.0;
                P = make_float4(INFINITY, INFINITY, INFINITY, 0.f);
            }
        };

        // 1) seed from the contiguous SFC window around the tile (Full / range mode), or around
        //    each query of a sparse tile of ascending centre indices (RandomSubset)
        i64 t0 = 0, t1 = -1;
        if (seed_base >= 0) {
            t0 = seed_base + static_cast<i64>(tile * 32);
            t1 = seed_base + static_cast<i64>(min(q.m, tile * 32 + 32));
        } else if (seed_base == kSeedSortedIdx) {
            t0 = q.idx[tile * 32];
            t1 = static_cast<i64>(q.idx[min(q.m, tile * 32 + 32) - 1]) + 1;
            if (t1 - t0 > 4 * 32 || t1 <= t0) {  // spread out (or unsorted: caller's order)
                t1 = -1;
                // per query: its own window, offered to it alone
                for (u32 am = act; am;) {
                    const int L = __ffs(am) - 1;
                    am &= am - 1;
                    const i64 c = q.idx[tile * 32 + L];
                    i64 lo = c - static_cast<i64>(seed_half / 2);
                    if (lo < 0) lo = 0;
                    i64 hi_ = lo + static_cast<i64>(seed_half);
                    if (hi_ > static_cast<i64>(npoints)) {
                        hi_ = static_cast<i64>(npoints);
                        lo = hi_ - static_cast<i64>(seed_half) < 0 ? 0 : hi_ - static_cast<i64>(seed_half);
                    }
                    for (i64 b = lo; b < hi_; b += 32) {
                        const bool valid = b + lane < hi_;
                        const u32 g = static_cast<u32>(b + lane);
                        float4 P;
                        double pd[3];
                        load_cand(valid, g, P, pd);
                        kw_buffer<R>(S, LD, LI, k, valid, g, P, pd, 1u << L, false, ext, E, lane);
                    }
                    if (lane == 0) S.sklo[L] = static_cast<u32>(lo), S.skhi[L] = static_cast<u32>(hi_);
                    __syncwarp();
                }
            }
        }
        if (t1 >= 0) {
            i64 lo = t0 - static_cast<i64>(seed_half);
            if (lo < 0) lo = 0;
            i64 hi_ = t1 + static_cast<i64>(seed_half);
            if (hi_ > static_cast<i64>(npoints)) hi_ = static_cast<i64>(npoints);
            for (i64 b = lo; b < hi_; b += 32) {
                const bool valid = b + lane < hi_;
                const u32 g = static_cast<u32>(b + lane);
                float4 P;
                double pd[3];
                load_cand(valid, g, P, pd);
                kw_buffer<R>(S, LD, LI, k, valid, g, P, pd, act, false, ext, E, lane);
            }
            S.sklo[lane] = static_cast<u32>(lo);
            S.skhi[lane] = static_cast<u32>(hi_);
            __syncwarp();
        }

        // 2) octree walk: a node is entered if some query's node threshold reaches its box; leaf
        //    points are gathered 32 at a time and offered to the queries that reach their leaves
        u32 fill = 0, qmask = 0;
        auto flush = [&]() {
            const bool valid = static_cast<u32>(lane) < fill;
            const u32 g = valid ? S.sidx[lane] : 0u;
            float4 P;
            double pd[3];
            load_cand(valid, g, P, pd);
            kw_buffer<R>(S, LD, LI, k, valid, g, P, pd, qmask, true, ext, E, lane);
            fill = 0;
            qmask = 0;
        };
        int sp = 1;
        if (lane == 0) S.stack[0] = 0;
        __syncwarp();
        while (sp > 0) {
            const u32 t = S.stack[--sp];
            const NodeF nd = load_node_f(tf, t);
            if (nd.nchild != 0) {
                bool keep = false;
                if (cl < static_cast<int>(nd.nchild)) {
                    const NodeF ch = load_node_f(tf, nd.child0 + cl);
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const float4 qq = S.qf[8 * grp + j];
                        const float nx = fmaxf(fmaxf(ch.lo[0] - qq.x, qq.x - ch.hi[0]), 0.f);
                        const float ny = fmaxf(fmaxf(ch.lo[1] - qq.y, qq.y - ch.hi[1]), 0.f);
                        const float nz = fmaxf(fmaxf(ch.lo[2] - qq.z, qq.z - ch.hi[2]), 0.f);
                        keep |= fmaf(nz, nz, fmaf(ny, ny, nx * nx)) <= S.tg[8 * grp + j];
                    }
                }
                u32 s = __ballot_sync(~0u, keep);
                s = (s | (s >> 8) | (s >> 16) | (s >> 24)) & 0xffu;
                const int kk = __popc(s);
                __syncwarp();
                if (lane < 8 && ((s >> lane) & 1u))
                    S.stack[sp + kk - 1 - __popc(s & ((1u << lane) - 1u))] = nd.child0 + lane;
                sp += kk;
                __syncwarp();
                continue;
            }
            bool want = false;
            if (active && (nd.begin < S.sklo[lane] || nd.end > S.skhi[lane])) {  // not wholly seeded
                const float nx = fmaxf(fmaxf(nd.lo[0] - qf.x, qf.x - nd.hi[0]), 0.f);
                const float ny = fmaxf(fmaxf(nd.lo[1] - qf.y, qf.y - nd.hi[1]), 0.f);
                const float nz = fmaxf(fmaxf(nd.lo[2] - qf.z, qf.z - nd.hi[2]), 0.f);
                want = fmaf(nz, nz, fmaf(ny, ny, nx * nx)) <= S.tg[lane];
            }
            const u32 wm = __ballot_sync(~0u, want);
            if (!wm) continue;
            for (u32 b = nd.begin; b < nd.end;) {
                const u32 take = min(32u - fill, nd.end - b);
                __syncwarp();
                if (static_cast<u32>(lane) < take) S.sidx[fill + lane] = b + lane;
                fill += take;
                qmask |= wm;
                b += take;
                if (fill == 32) {
                    __syncwarp();
                    flush();
                }
            }
        }
        if (fill) {
            __syncwarp();
            flush();
        }
        __syncwarp();

        // 3) the lists are sorted: coalesced row writes
        const u64 left = q.m - tile * 32;
        const u32 nact = left < 32 ? static_cast<u32>(left) : 32u;
        for (u32 L = 0; L < nact; ++L) {
            const u64 row = tile * 32 + L;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const u32 p = lane + 32 * r;
                if (p < k) {
                    out_idx[row * k + p] = LI[static_cast<u64>(L) * k + p];
                    out_dist[row * k + p] = LD[static_cast<u64>(L) * k + p];
                }
            }
        }
        __syncwarp();
    }
}

inline size_t knn_warp_smem_per_warp(u32 k) {
    return (sizeof(KwShared) + 15) / 16 * 16 + static_cast<size_t>(32) * k * 12;
}

}  // namespace lo
