// knn.cu -- K7 exact kNN over the octree, K8 kNN row digests, K9 locality histogram.
//
// Replaces knn_lin_oct / run_knn_batch (search.cpp:158-259, :369-388) and the locality
// accumulation (locality.cpp:41-97).  The reference's best-first queue emits the first k
// points of the whole cloud under the order (dist_sq, index); this kernel computes the same
// set with a warp-shared depth-first walk: one warp owns 32 consecutive queries, children are
// visited nearest-first (distance from the tile's mean query to the child's box), and each
// lane keeps a bounded max-heap of its k best (dist_sq, index) pairs.  A lane skips a node
// only when its heap is full and the box's lower bound is strictly greater than its current
// worst distance, so equal-distance points with a lower index are never lost.
#include <algorithm>
#include <cmath>

#include "search_common.cuh"

namespace lo {

u32* upload_centres(lo_context* ctx, const u32* centres_host, u64 m, u64 n);
void upload_points(lo_context* ctx, const lo_coded* c, const double* xyz_host, u64 m, double** x,
                   double** y, double** z, float4** f, double* bmax);

// (a.d, a.i) > (b.d, b.i) lexicographically: heap_after (search.cpp:173-177) on points.
__device__ __forceinline__ bool after(double ad, u32 ai, double bd, u32 bi) {
    return ad > bd || (ad == bd && ai > bi);
}

// Max-heap of one lane; element e lives at hd[e * 32] / hi[e * 32] (lane-interleaved).
struct LaneHeap {
    double* hd;
    u32* hi;
    u32 size;

    __device__ __forceinline__ bool after(double a, u32 ia, double b, u32 ib) const {
        return lo::after(a, ia, b, ib);
    }

    __device__ __forceinline__ void push(double d, u32 i) {
        u32 pos = size++;
        while (pos > 0) {
            const u32 par = (pos - 1) >> 1;
            const double pd = hd[par * 32];
            const u32 pi = hi[par * 32];
            if (!after(d, i, pd, pi)) break;
            hd[pos * 32] = pd;
            hi[pos * 32] = pi;
            pos = par;
        }
        hd[pos * 32] = d;
        hi[pos * 32] = i;
    }

    // sift_down for a compile-time n = 2^LOGK: at most LOGK levels, fully unrolled
    template <int LOGK>
    __device__ __forceinline__ void sift_down_fixed(double d, u32 i) {
        constexpr u32 n = 1u << LOGK;
        u32 pos = 0;
#pragma unroll
        for (int lv = 0; lv < LOGK; ++lv) {
            u32 c = 2 * pos + 1;
            if (c >= n) break;
            double cd = hd[c * 32];
            u32 ci = hi[c * 32];
            if (c + 1 < n) {
                const double rd = hd[(c + 1) * 32];
                const u32 ri = hi[(c + 1) * 32];
                if (after(rd, ri, cd, ci)) {
                    c = c + 1;
                    cd = rd;
                    ci = ri;
                }
            }
            if (!after(cd, ci, d, i)) break;
            hd[pos * 32] = cd;
            hi[pos * 32] = ci;
            pos = c;
        }
        hd[pos * 32] = d;
        hi[pos * 32] = i;
    }

    // replace the maximum and restore the heap over [0, n)
    __device__ __forceinline__ void sift_down(double d, u32 i, u32 n) {
        u32 pos = 0;
        for (;;) {
            u32 c = 2 * pos + 1;
            if (c >= n) break;
            double cd = hd[c * 32];
            u32 ci = hi[c * 32];
            if (c + 1 < n) {
                const double rd = hd[(c + 1) * 32];
                const u32 ri = hi[(c + 1) * 32];
                if (after(rd, ri, cd, ci)) {
                    c = c + 1;
                    cd = rd;
                    ci = ri;
                }
            }
            if (!after(cd, ci, d, i)) break;
            hd[pos * 32] = cd;
            hi[pos * 32] = ci;
            pos = c;
        }
        hd[pos * 32] = d;
        hi[pos * 32] = i;
    }
};

constexpr int kKnnSmemBudget = 200 * 1024;

}  // namespace lo

#include "knn_float.cuh"
#include "knn_warp.cuh"
#include "knn_select.cuh"

namespace lo {

template <bool GLOBAL_HEAP>
__global__ void __launch_bounds__(128) knn_kernel(const TNode* __restrict__ tn,
                                                  const double* __restrict__ px,
                                                  const double* __restrict__ py,
                                                  const double* __restrict__ pz, Queries q, u32 k,
                                                  u32 keff, u32* __restrict__ out_idx,
                                                  double* __restrict__ out_dist,
                                                  double* __restrict__ gheap_d,
                                                  u32* __restrict__ gheap_i) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int warps = blockDim.x >> 5;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    // shared layout: [stack: warps * kStackCap u32][sx, sy, sz: warps * 32 f64 each][heaps]
    u32* stack = reinterpret_cast<u32*>(smem) + w * kStackCap;
    double* stage = reinterpret_cast<double*>(smem + sizeof(u32) * kStackCap * warps);
    double* sx = stage + w * 96;
    double* sy = sx + 32;
    double* sz = sy + 32;
    double* hd;
    u32* hi;
    if (GLOBAL_HEAP) {
        const u64 slot = static_cast<u64>(blockIdx.x) * warps + w;
        hd = gheap_d + slot * k * 32 + lane;
        hi = gheap_i + slot * k * 32 + lane;
    } else {
        double* heaps_d = stage + warps * 96;
        u32* heaps_i = reinterpret_cast<u32*>(heaps_d + static_cast<u64>(warps) * k * 32);
        hd = heaps_d + static_cast<u64>(w) * k * 32 + lane;
        hi = heaps_i + static_cast<u64>(w) * k * 32 + lane;
    }
    const u64 ntiles = (q.m + 31) / 32;
    for (u64 tile = static_cast<u64>(blockIdx.x) * warps + w; tile < ntiles;
         tile += static_cast<u64>(gridDim.x) * warps) {
        const u64 qi = tile * 32 + lane;
        const bool active = qi < q.m;
        double cx = 0.0, cy = 0.0, cz = 0.0;
        if (active) load_query(q, qi, cx, cy, cz);
        // warp anchor for the child visiting order: mean of the active queries
        double ax = active ? cx : 0.0, ay = active ? cy : 0.0, az = active ? cz : 0.0;
        const int nact = __popc(__ballot_sync(~0u, active));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            ax += __shfl_xor_sync(~0u, ax, o);
            ay += __shfl_xor_sync(~0u, ay, o);
            az += __shfl_xor_sync(~0u, az, o);
        }
        ax /= nact, ay /= nact, az /= nact;
        LaneHeap heap{hd, hi, 0};
        double worst_d = 0.0;
        u32 worst_i = 0;
        int sp = 1;
        if (lane == 0) stack[0] = 0;
        __syncwarp();
        while (sp > 0) {
            const u32 t = stack[--sp];
            const NodeView nd = load_node(tn, t);
            bool visit = false;
            if (active) visit = heap.size < k || box_dist_sq(cx, cy, cz, nd) <= worst_d;
            if (!__any_sync(~0u, visit)) continue;
            if (nd.nchild == 0) {
                for (u32 base = nd.begin; base < nd.end; base += 32) {
                    const u32 j = base + lane;
                    __syncwarp();
                    if (j < nd.end) {
                        sx[lane] = px[j];
                        sy[lane] = py[j];
                        sz[lane] = pz[j];
                    }
                    __syncwarp();
                    if (visit) {
                        const u32 cnt = min(32u, nd.end - base);
                        for (u32 jj = 0; jj < cnt; ++jj) {
                            const double d = point_dist_sq(sx[jj], sy[jj], sz[jj], cx, cy, cz);
                            const u32 id = base + jj;
                            if (heap.size < k) {
                                heap.push(d, id);
                                if (heap.size == k) {
                                    worst_d = hd[0];
                                    worst_i = hi[0];
                                }
                            } else if (after(worst_d, worst_i, d, id)) {
                                heap.sift_down(d, id, k);
                                worst_d = hd[0];
                                worst_i = hi[0];
                            }
                        }
                    }
                }
            } else {
                // nearest-first: rank children by (box distance to the anchor, code order)
                double cd = 0.0;
                const u32 nc = nd.nchild;
                if (lane < static_cast<int>(nc)) cd = box_dist_sq(ax, ay, az, load_node(tn, nd.child0 + lane));
                u32 rank = 0;
                for (u32 o = 0; o < nc; ++o) {
                    const double od = __shfl_sync(~0u, cd, o);
                    if (od < cd || (od == cd && static_cast<int>(o) < lane)) ++rank;
                }
                __syncwarp();
                if (lane < static_cast<int>(nc)) stack[sp + nc - 1 - rank] = nd.child0 + lane;
                sp += nc;
                __syncwarp();
            }
        }
        if (active) {
            // heap sort in place -> ascending (dist_sq, index), then write the row
            const u32 n = heap.size;
            for (u32 e = n; e > 1; --e) {
                const double td = hd[0];
                const u32 ti = hi[0];
                const double ld = hd[(e - 1) * 32];
                const u32 li = hi[(e - 1) * 32];
                hd[(e - 1) * 32] = td;
                hi[(e - 1) * 32] = ti;
                heap.sift_down(ld, li, e - 1);
            }
            u32* oi = out_idx + qi * keff;
            double* od = out_dist + qi * keff;
            for (u32 e = 0; e < n; ++e) {
                oi[e] = hi[e * 32];
                od[e] = hd[e * 32];
            }
        }
        __syncwarp();
    }
}

// FNV-1a-64 of (index, bit pattern of dist_sq) pairs (search.cpp:376-381).
__global__ void knn_digest(const u32* __restrict__ idx, const double* __restrict__ dist, u64 m,
                           u32 keff, u64* __restrict__ fps) {
    for (u64 r = blockIdx.x * (u64)blockDim.x + threadIdx.x; r < m;
         r += (u64)gridDim.x * blockDim.x) {
        u64 h = kFnvOffset;
        for (u32 j = 0; j < keff; ++j) {
            h = fnv_u32(h, idx[r * keff + j]);
            h = fnv_u64(h, static_cast<u64>(__double_as_longlong(dist[r * keff + j])));
        }
        fps[r] = h;
    }
}

// K9: log2-binned |map(i) - map(j)| over every (centre, neighbour) pair (locality.cpp:41-87).
__global__ void locality_kernel(const u32* __restrict__ idx, u64 m, u32 keff,
                                const u32* __restrict__ centres, const u32* __restrict__ map,
                                unsigned long long* __restrict__ bins) {
    __shared__ unsigned long long sb[33];
    if (threadIdx.x < 33) sb[threadIdx.x] = 0;
    __syncthreads();
    for (u64 e = blockIdx.x * (u64)blockDim.x + threadIdx.x; e < m * keff;
         e += (u64)gridDim.x * blockDim.x) {
        const u64 r = e / keff;
        const u32 ci = centres ? centres[r] : static_cast<u32>(r);
        const u64 mi = map ? map[ci] : ci;
        const u64 mj = map ? map[idx[e]] : idx[e];
        const u64 d = mi > mj ? mi - mj : mj - mi;
        const int b = d == 0 ? 0 : 64 - __clzll(static_cast<long long>(d));
        atomicAdd(&sb[b], 1ull);
    }
    __syncthreads();
    if (threadIdx.x < 33 && sb[threadIdx.x]) atomicAdd(&bins[threadIdx.x], sb[threadIdx.x]);
}

// Exact locality histogram (locality.cpp:41-97): count of every |map(i) - map(j)| into a dense
// u64 array over d in [0, n); small d (the bulk for SFC orders) goes through a per-block
// shared-memory histogram first, so the hot bins see no global atomic contention.
constexpr u32 kLocSmall = 4096;
__global__ void locality_dense(const u32* __restrict__ idx, u64 m, u32 keff,
                               const u32* __restrict__ centres, const u32* __restrict__ map,
                               unsigned long long* __restrict__ dense) {
    __shared__ u32 sh[kLocSmall];
    for (u32 i = threadIdx.x; i < kLocSmall; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    for (u64 e = blockIdx.x * (u64)blockDim.x + threadIdx.x; e < m * keff;
         e += (u64)gridDim.x * blockDim.x) {
        const u64 r = e / keff;
        const u32 ci = centres ? centres[r] : static_cast<u32>(r);
        const u32 mi = map ? map[ci] : ci;
        const u32 mj = map ? map[idx[e]] : idx[e];
        const u32 d = mi > mj ? mi - mj : mj - mi;
        if (d < kLocSmall) atomicAdd(&sh[d], 1u);
        else atomicAdd(&dense[d], 1ull);
    }
    __syncthreads();
    for (u32 i = threadIdx.x; i < kLocSmall; i += blockDim.x)
        if (sh[i]) atomicAdd(&dense[i], static_cast<unsigned long long>(sh[i]));
}

// Sparse path (index maps whose value span exceeds the dense array): every pair's d as a u64
// key, then sort + run-length encode.
__global__ void locality_pairs(const u32* __restrict__ idx, u64 m, u32 keff, const u32* __restrict__ centres,
                               const u32* __restrict__ map, u64* __restrict__ keys, u32* __restrict__ hist) {
    __shared__ u32 h[4 * 256];
    for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) h[i] = 0;
    __syncthreads();
    for (u64 e = blockIdx.x * (u64)blockDim.x + threadIdx.x; e < m * keff; e += (u64)gridDim.x * blockDim.x) {
        const u64 r = e / keff;
        const u32 ci = centres ? centres[r] : static_cast<u32>(r);
        const u32 mi = map[ci], mj = map[idx[e]];
        const u32 d = mi > mj ? mi - mj : mj - mi;
        keys[e] = d;
#pragma unroll
        for (int b = 0; b < 4; ++b) atomicAdd(&h[b * 256 + ((d >> (8 * b)) & 0xffu)], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x)
        if (h[i]) atomicAdd(&hist[i], h[i]);
}

__global__ void run_heads(const u64* __restrict__ ks, u64 n, u32* __restrict__ f) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        f[i] = i == 0 || ks[i] != ks[i - 1];
}

__global__ void run_emit(const u64* __restrict__ ks, const u64* __restrict__ pos, u64 n, u32* __restrict__ d_out,
                         u64* __restrict__ start) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        if (i == 0 || ks[i] != ks[i - 1]) {
            d_out[pos[i]] = static_cast<u32>(ks[i]);
            start[pos[i]] = i;
        }
}

__global__ void run_lengths(const u64* __restrict__ start, u64 nb, u64 n, u64* __restrict__ c_out) {
    for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < nb; j += (u64)gridDim.x * blockDim.x)
        c_out[j] = (j + 1 < nb ? start[j + 1] : n) - start[j];
}

__global__ void nonzero_flags(const unsigned long long* __restrict__ dense, u64 n, u32* __restrict__ f) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        f[i] = dense[i] != 0;
}

__global__ void compact_bins(const unsigned long long* __restrict__ dense, const u64* __restrict__ pos,
                             u64 n, u32* __restrict__ d_out, u64* __restrict__ c_out) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const unsigned long long c = dense[i];
        if (c) {
            d_out[pos[i]] = static_cast<u32>(i);
            c_out[pos[i]] = c;
        }
    }
}

// seed_base >= 0: query i is cloud point seed_base + i (Full / range mode), which lets each
// tile seed its heaps from the contiguous SFC window around it.
static lo_knn_result* knn_search(lo_context* ctx, const lo_octree* t, const lo_coded* c, u32 k,
                                 const Queries& q, bool fingerprint, i64 seed_base) {
    require(t != nullptr && c != nullptr, LO_INVALID_ARGUMENT, "null tree or cloud");
    require(k >= 1, LO_INVALID_ARGUMENT, "knn: k must be >= 1");
    auto* out = new lo_knn_result;
    out->ctx = ctx;
    out->rows = q.m;
    out->k = k;
    out->keff = static_cast<u32>(std::min<u64>(k, c->n));
    // the heap never holds more than N entries, so k > N behaves as k = N
    const u32 kh = out->keff;
    cudaEvent_t e0, e1;
    LO_CUDA(cudaEventCreate(&e0));
    LO_CUDA(cudaEventCreate(&e1));
    double* gd = nullptr;
    float* gk = nullptr;
    u32* gi = nullptr;
    try {
        LO_CUDA(cudaEventRecord(e0, ctx->stream));
        out->idx = dalloc_t<u32>(ctx, q.m * kh);
        out->dist = dalloc_t<double>(ctx, q.m * kh);
        const bool use_float = q.f && t->tf && c->pf && !force_fp64();
        // FP32-filtered kernel: (key f32, index) heap entries; exact fallback: (f64, index)
        const bool keyed = use_float && kh >= 32;  // compact heap entries where occupancy binds
        const size_t per_warp_heap = static_cast<size_t>(kh) * 32 * (keyed ? 8 : 12);
        const size_t per_warp_fixed =
            use_float ? kKnnFixed : sizeof(u32) * kStackCap + 96 * sizeof(double);
        const bool global_heap = per_warp_heap + per_warp_fixed > static_cast<size_t>(kKnnSmemBudget);
        // warps per block: the most resident warps per SM under the shared-memory budget
        int warps = 4;
        if (!global_heap) {
            int best = 0;
            for (int w = 4; w >= 1; w >>= 1) {
                const size_t blk = w * (per_warp_heap + per_warp_fixed);
                if (blk > static_cast<size_t>(kKnnSmemBudget)) continue;
                const int resident = w * std::min(16, static_cast<int>(220 * 1024 / blk));
                if (resident > best) best = resident, warps = w;
            }
        }
        const size_t smem = warps * (per_warp_fixed + (global_heap ? 0 : per_warp_heap));
        int per_sm = std::max(1, static_cast<int>(220 * 1024 / std::max<size_t>(smem, 1)));
        per_sm = std::min(per_sm, 16);
        auto grid_for = [&](u64 rows) {
            const u64 tl = (rows + 31) / 32;
            return static_cast<int>(std::max<u64>(
                1, std::min<u64>((tl + warps - 1) / warps, static_cast<u64>(ctx->sm_count) * per_sm)));
        };
        const u64 tiles = (q.m + 31) / 32;
        const int blocks = grid_for(q.m);
        float E = static_cast<float>(std::ldexp(std::max(c->bmax, q.bmax), -23));
        E = std::nextafter(E, INFINITY);  // round up
        // the FP32-filtered heap kernel over queries qq, rows into (oi, od)
        auto launch_heaps = [&](const Queries& qq, i64 sb, u32* oi, double* od) {
            const int hb = grid_for(qq.m);
            const u32 seed_half = std::max<u32>(16, kh);
            u64* counter = dalloc_t<u64>(ctx, 1);
            LO_CUDA(cudaMemsetAsync(counter, 0, 8, ctx->stream));
            if (global_heap) {
                if (!gk) {
                    gk = dalloc_t<float>(ctx, static_cast<u64>(blocks) * warps * kh * 32);
                    gi = dalloc_t<u32>(ctx, static_cast<u64>(blocks) * warps * kh * 32);
                }
                LO_CUDA(cudaFuncSetAttribute(knn_float_kernel<true, 0, true>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
                knn_float_kernel<true, 0, true><<<std::min(hb, blocks), 32 * warps, smem, ctx->stream>>>(
                    t->tf, c->pf, c->x, c->y, c->z, c->n, qq, sb, seed_half, E, kh, oi, od, gk, gi, counter);
            } else {
                // common k compile to fixed-depth, unrolled heap sifts
#define LO_KNN_LAUNCH(KC, KEYED)                                                                          \
    do {                                                                                                  \
        LO_CUDA(cudaFuncSetAttribute(knn_float_kernel<false, KC, KEYED>,                                  \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));\
        knn_float_kernel<false, KC, KEYED><<<hb, 32 * warps, smem, ctx->stream>>>(                        \
            t->tf, c->pf, c->x, c->y, c->z, c->n, qq, sb, seed_half, E, kh, oi, od, nullptr, nullptr,     \
            counter);                                                                                     \
    } while (0)
                switch (kh) {
                    case 8: LO_KNN_LAUNCH(8, false); break;
                    case 16: LO_KNN_LAUNCH(16, false); break;
                    case 32: LO_KNN_LAUNCH(32, true); break;
                    case 64: LO_KNN_LAUNCH(64, true); break;
                    default:
                        if (keyed) LO_KNN_LAUNCH(0, true);
                        else LO_KNN_LAUNCH(0, false);
                        break;
                }
#undef LO_KNN_LAUNCH
            }
            LO_CHECK_LAUNCH();
            dfree(ctx, counter);
        };
        stage_begin(ctx, "knn");
        // LO_KNN_WARP=1: the warp-cooperative kernel (knn_warp.cuh, k <= 64).  Exact, but measured 4-6x
        // slower than the per-lane heaps (cfg1 k = 8/16/32/64: 31.9/44.6/120/386 vs 6.6/11.0/21.6/59.6 ms):
        // every insertion is a warp-wide shuffle chain serialised per query, and the seed window offers
        // ~k candidates to each of the 32 queries one query at a time (the per-lane heaps take them in
        // parallel).  Kept as the measured alternative; DESIGN.md §8.
        const bool warp_kernel = use_float && kh <= 64 && env_flag("LO_KNN_WARP");
        // LO_KNN_SELECT=1: candidate collection + warp selection (knn_select.cuh) for batches of cloud
        // points (Full / range / centre lists)
        const bool select_path = use_float && kh <= 64 && seed_base != -1 && env_flag("LO_KNN_SELECT");
        if (q.m && warp_kernel) {
            const u32 seed_half = std::max<u32>(16, kh);
            const size_t per_warp = knn_warp_smem_per_warp(kh);
            const size_t wsmem = kKwWarps * per_warp;
            const int wper_sm = std::max(1, std::min(16, static_cast<int>(224 * 1024 / wsmem)));
            const int wblocks = static_cast<int>(std::max<u64>(
                1, std::min<u64>((tiles + kKwWarps - 1) / kKwWarps, static_cast<u64>(ctx->sm_count) * wper_sm)));
            u64* counter = dalloc_t<u64>(ctx, 1);
            LO_CUDA(cudaMemsetAsync(counter, 0, 8, ctx->stream));
            if (kh <= 32) {
                ensure_smem_attr(ctx, kAttrKnnW1, knn_warp_kernel<1>, kKwWarps * knn_warp_smem_per_warp(32));
                knn_warp_kernel<1><<<wblocks, 32 * kKwWarps, wsmem, ctx->stream>>>(
                    t->tf, c->x, c->y, c->z, c->n, q, seed_base, seed_half, E, kh, out->idx, out->dist, counter);
            } else {
                ensure_smem_attr(ctx, kAttrKnnW2, knn_warp_kernel<2>, kKwWarps * knn_warp_smem_per_warp(64));
                knn_warp_kernel<2><<<wblocks, 32 * kKwWarps, wsmem, ctx->stream>>>(
                    t->tf, c->x, c->y, c->z, c->n, q, seed_base, seed_half, E, kh, out->idx, out->dist, counter);
            }
            LO_CHECK_LAUNCH();
            dfree(ctx, counter);
        } else if (q.m && select_path) {
            knn_select_run(ctx, t, c, q, kh, seed_base, E, out->idx, out->dist, launch_heaps);
        } else if (q.m && use_float) {
            launch_heaps(q, seed_base, out->idx, out->dist);
        } else if (q.m) {
            if (global_heap) {
                gd = dalloc_t<double>(ctx, static_cast<u64>(blocks) * warps * kh * 32);
                gi = dalloc_t<u32>(ctx, static_cast<u64>(blocks) * warps * kh * 32);
                LO_CUDA(cudaFuncSetAttribute(knn_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem)));
                knn_kernel<true><<<blocks, 32 * warps, smem, ctx->stream>>>(
                    t->tn, c->x, c->y, c->z, q, kh, kh, out->idx, out->dist, gd, gi);
            } else {
                LO_CUDA(cudaFuncSetAttribute(knn_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem)));
                knn_kernel<false><<<blocks, 32 * warps, smem, ctx->stream>>>(
                    t->tn, c->x, c->y, c->z, q, kh, kh, out->idx, out->dist, nullptr, nullptr);
            }
            LO_CHECK_LAUNCH();
        }
        stage_end(ctx);
        if (fingerprint) {
            out->fps = dalloc_t<u64>(ctx, q.m);
            if (q.m) {
                knn_digest<<<std::max(1, ceil_div(q.m, 256)), 256, 0, ctx->stream>>>(
                    out->idx, out->dist, q.m, kh, out->fps);
                LO_CHECK_LAUNCH();
            }
        }
        LO_CUDA(cudaEventRecord(e1, ctx->stream));
        sync(ctx);
        LO_CUDA(cudaEventElapsedTime(&out->ms, e0, e1));
    } catch (...) {
        dfree(ctx, out->idx);
        dfree(ctx, out->dist);
        dfree(ctx, out->fps);
        dfree(ctx, gd);
        dfree(ctx, gk);
        dfree(ctx, gi);
        delete out;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        throw;
    }
    dfree(ctx, gd);
    dfree(ctx, gk);
    dfree(ctx, gi);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return out;
}

}  // namespace lo

using namespace lo;

extern "C" {

int lo_knn(lo_context* ctx, const lo_octree* tree, const lo_coded* coded, uint32_t k,
           const uint32_t* centres_host, uint64_t m, int fingerprint, lo_knn_result** out) {
    return api_ctx(ctx, [&] {
        require(k >= 1, LO_INVALID_ARGUMENT, "knn: k must be >= 1");
        require(tree && coded, LO_INVALID_ARGUMENT, "null tree or cloud");
        const u64 rows = centres_host ? m : coded->n;
        ensure_float_shadows(ctx, coded, tree);
        u32* cidx = upload_centres(ctx, centres_host, m, coded->n);
        // explicit centres are searched in curve order, rows scattered back (centres.cu)
        const bool sorted = centres_host && ctx->centre_sort;  // LO_OPT_CENTRE_ORDER
        SortedCentres sc = sort_centres(ctx, cidx, sorted ? m : 0);
        Queries q{coded->x, coded->y, coded->z, centres_host ? (sorted ? sc.idx : cidx) : nullptr, rows, coded->pf,
                  coded->bmax};
        try {
            *out = knn_search(ctx, tree, coded, k, q, fingerprint != 0, centres_host ? kSeedSortedIdx : 0);
            if (sorted) unsort_knn(ctx, sc, *out);
        } catch (...) {
            dfree(ctx, cidx), dfree(ctx, sc.idx), dfree(ctx, sc.pos);
            throw;
        }
        dfree(ctx, cidx), dfree(ctx, sc.idx), dfree(ctx, sc.pos);
    });
}

int lo_knn_points(lo_context* ctx, const lo_octree* tree, const lo_coded* coded, uint32_t k,
                  const double* queries_host, uint64_t m, lo_knn_result** out) {
    return api_ctx(ctx, [&] {
        require(k >= 1, LO_INVALID_ARGUMENT, "knn: k must be >= 1");
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
            *out = knn_search(ctx, tree, coded, k, q, true, -1);
            unsort_knn(ctx, sc, *out);
        } catch (...) {
            dfree(ctx, x), dfree(ctx, y), dfree(ctx, z), dfree(ctx, f), dfree(ctx, sc.pos);
            throw;
        }
        dfree(ctx, x), dfree(ctx, y), dfree(ctx, z), dfree(ctx, f), dfree(ctx, sc.pos);
    });
}

int lo_knn_range(lo_context* ctx, const lo_octree* tree, const lo_coded* coded, uint32_t k,
                 uint64_t begin, uint64_t end, int fingerprint, lo_knn_result** out) {
    return api_ctx(ctx, [&] {
        require(k >= 1, LO_INVALID_ARGUMENT, "knn: k must be >= 1");
        require(tree && coded, LO_INVALID_ARGUMENT, "null tree or cloud");
        require(begin <= end && end <= coded->n, LO_INVALID_ARGUMENT, "centre range out of bounds");
        ensure_float_shadows(ctx, coded, tree);
        Queries q{coded->x + begin, coded->y + begin, coded->z + begin, nullptr, end - begin,
                  coded->pf + begin, coded->bmax};
        *out = knn_search(ctx, tree, coded, k, q, fingerprint != 0, static_cast<i64>(begin));
    });
}

int lo_knn_info_get(const lo_knn_result* res, uint64_t* rows, uint32_t* k_eff, double* device_ms) {
    return api([&] {
        if (rows) *rows = res->rows;
        if (k_eff) *k_eff = res->keff;
        if (device_ms) *device_ms = res->ms;
    });
}

int lo_knn_download(lo_context* ctx, const lo_knn_result* res, uint32_t* idx_host, double* dist_host,
                    uint64_t* fingerprints_host) {
    return api_ctx(ctx, [&] {
        const u64 e = res->rows * res->keff;
        if (idx_host && e)
            LO_CUDA(cudaMemcpyAsync(idx_host, res->idx, 4 * e, cudaMemcpyDeviceToHost, ctx->stream));
        if (dist_host && e)
            LO_CUDA(cudaMemcpyAsync(dist_host, res->dist, 8 * e, cudaMemcpyDeviceToHost, ctx->stream));
        if (fingerprints_host && res->rows) {
            require(res->fps != nullptr, LO_INVALID_ARGUMENT, "fingerprints were not computed");
            LO_CUDA(cudaMemcpyAsync(fingerprints_host, res->fps, 8 * res->rows,
                                    cudaMemcpyDeviceToHost, ctx->stream));
        }
        sync(ctx);
    });
}

// Same as lo_knn_download, asynchronously on the context's copy stream (pinned host buffers):
// the next batch computes while these rows travel; the result may be destroyed before the
// copy lands (its buffers are released behind it).
int lo_knn_download_async(lo_context* ctx, lo_knn_result* res, uint32_t* idx_host, double* dist_host,
                          uint64_t* fingerprints_host) {
    return api_ctx(ctx, [&] {
        require(res != nullptr, LO_INVALID_ARGUMENT, "null result");
        require(!fingerprints_host || !res->rows || res->fps, LO_INVALID_ARGUMENT, "fingerprints were not computed");
        if (!res->copied) LO_CUDA(cudaEventCreateWithFlags(&res->copied, cudaEventDisableTiming));
        cudaEvent_t ready;
        LO_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
        LO_CUDA(cudaEventRecord(ready, ctx->stream));
        LO_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ready, 0));
        cudaEventDestroy(ready);  // released once the recorded work completes
        const cudaStream_t s = ctx->copy_stream;
        const u64 e = res->rows * res->keff;
        if (idx_host && e) LO_CUDA(cudaMemcpyAsync(idx_host, res->idx, 4 * e, cudaMemcpyDeviceToHost, s));
        if (dist_host && e) LO_CUDA(cudaMemcpyAsync(dist_host, res->dist, 8 * e, cudaMemcpyDeviceToHost, s));
        if (fingerprints_host && res->rows)
            LO_CUDA(cudaMemcpyAsync(fingerprints_host, res->fps, 8 * res->rows, cudaMemcpyDeviceToHost, s));
        LO_CUDA(cudaEventRecord(res->copied, s));
    });
}

int lo_knn_destroy(lo_knn_result* res) {
    if (!res) return LO_OK;
    return api_ctx(res->ctx, [&] {
        lo_context* ctx = res->ctx;
        bool pending = false;
        if (res->copied) {
            pending = cudaEventQuery(res->copied) != cudaSuccess;
            if (pending) cudaGetLastError();  // cudaErrorNotReady is not an error
            cudaEventDestroy(res->copied);
        }
        if (pending) {  // an async download still reads them: release behind the copy stream
            big_release(ctx, res->idx, 0, ctx->copy_stream);
            big_release(ctx, res->dist, 0, ctx->copy_stream);
            big_release(ctx, res->fps, 0, ctx->copy_stream);
        } else {
            dfree(ctx, res->idx);
            dfree(ctx, res->dist);
            dfree(ctx, res->fps);
        }
        delete res;
    });
}

int lo_locality_log2(lo_context* ctx, const lo_knn_result* res, const lo_coded* coded,
                     const uint32_t* centres_host, int use_perm, uint64_t* bins33_host) {
    return api_ctx(ctx, [&] {
        u32* cidx = upload_centres(ctx, centres_host, centres_host ? res->rows : 0, coded->n);
        unsigned long long* bins = dalloc_t<unsigned long long>(ctx, 33);
        LO_CUDA(cudaMemsetAsync(bins, 0, 33 * 8, ctx->stream));
        const u64 e = res->rows * res->keff;
        if (e)
            locality_kernel<<<std::max(1, std::min(ceil_div(e, 256), ctx->sm_count * 8)), 256, 0,
                              ctx->stream>>>(res->idx, res->rows, res->keff, cidx,
                                             use_perm ? coded->perm : nullptr, bins);
        LO_CHECK_LAUNCH();
        LO_CUDA(cudaMemcpyAsync(bins33_host, bins, 33 * 8, cudaMemcpyDeviceToHost, ctx->stream));
        dfree(ctx, bins);
        dfree(ctx, cidx);
        sync(ctx);
    });
}

int lo_locality_histogram(lo_context* ctx, const lo_knn_result* res, const lo_coded* coded,
                          const uint32_t* centres_host, const uint32_t* index_map_host,
                          uint64_t* nbins, uint32_t* d_host, uint64_t* count_host, uint64_t cap) {
    return api_ctx(ctx, [&] {
        require(res && coded && nbins, LO_INVALID_ARGUMENT, "null argument");
        const u64 n = coded->n;
        u32* cidx = upload_centres(ctx, centres_host, centres_host ? res->rows : 0, n);
        u32* map = nullptr;
        unsigned long long* dense = nullptr;
        u32* flags = nullptr;
        u64* pos = nullptr;
        u32* dd = nullptr;
        u64* cc = nullptr;
        auto release = [&] {
            dfree(ctx, cidx), dfree(ctx, map), dfree(ctx, dense), dfree(ctx, flags), dfree(ctx, pos);
            dfree(ctx, dd), dfree(ctx, cc);
        };
        try {
            // d = |map(i) - map(j)| < span of the map's values (any u32 is a legal map value,
            // locality.cpp:47-49): a dense array over [0, span) when that is small enough, else
            // sort + run-length encode the pairs' d
            u64 span = n;
            if (index_map_host && n) {
                const auto mm = std::minmax_element(index_map_host, index_map_host + n);
                span = static_cast<u64>(*mm.second) - *mm.first + 1;
            }
            if (index_map_host) {
                map = dalloc_t<u32>(ctx, n);
                LO_CUDA(cudaMemcpyAsync(map, index_map_host, 4 * n, cudaMemcpyHostToDevice, ctx->stream));
            }
            const u64 pairs = res->rows * res->keff;
            if (span > std::max<u64>(n, 1ull << 27)) {
                require(pairs < (1ull << 32), LO_INVALID_ARGUMENT,
                        "locality histogram: too many pairs for a sparse index map");
                u64* keys = dalloc_t<u64>(ctx, pairs);
                u64* ks = nullptr;
                u32* perm = nullptr;
                u32* hist = nullptr;
                u64* start = nullptr;
                try {
                    ks = dalloc_t<u64>(ctx, pairs);
                    perm = dalloc_t<u32>(ctx, pairs);
                    hist = dalloc_t<u32>(ctx, 4 * 256);
                    LO_CUDA(cudaMemsetAsync(hist, 0, 4 * 256 * 4, ctx->stream));
                    const int g = std::max(1, std::min(ceil_div(pairs, 256), ctx->sm_count * 8));
                    if (pairs) {
                        locality_pairs<<<g, 256, 0, ctx->stream>>>(res->idx, res->rows, res->keff, cidx, map, keys,
                                                                 hist);
                        LO_CHECK_LAUNCH();
                    }
                    std::vector<u32> hh(8 * 256, 0);
                    fetch_small(ctx, hist, 4 * 256 * 4);
                    std::memcpy(hh.data(), ctx->pinned_scratch, 4 * 256 * 4);
                    hh[4 * 256] = static_cast<u32>(pairs);  // bits 32..39 are zero
                    if (pairs) radix_sort(ctx, keys, pairs, hh.data(), 11, ks, perm);
                    flags = dalloc_t<u32>(ctx, pairs);
                    pos = dalloc_t<u64>(ctx, pairs + 1);
                    run_heads<<<g, 256, 0, ctx->stream>>>(ks, pairs, flags);
                    LO_CHECK_LAUNCH();
                    exclusive_scan_u32_to_u64(ctx, flags, pos, pairs);
                    const u64 nb = read_scalar(ctx, pos + pairs);
                    *nbins = nb;
                    if (d_host && count_host && nb <= cap && nb) {
                        dd = dalloc_t<u32>(ctx, nb);
                        cc = dalloc_t<u64>(ctx, nb);
                        start = dalloc_t<u64>(ctx, nb);
                        run_emit<<<g, 256, 0, ctx->stream>>>(ks, pos, pairs, dd, start);
                        LO_CHECK_LAUNCH();
                        run_lengths<<<std::max(1, std::min(ceil_div(nb, 256), ctx->sm_count * 8)), 256, 0,
                                      ctx->stream>>>(start, nb, pairs, cc);
                        LO_CHECK_LAUNCH();
                        LO_CUDA(cudaMemcpyAsync(d_host, dd, 4 * nb, cudaMemcpyDeviceToHost, ctx->stream));
                        LO_CUDA(cudaMemcpyAsync(count_host, cc, 8 * nb, cudaMemcpyDeviceToHost, ctx->stream));
                    }
                    sync(ctx);
                } catch (...) {
                    dfree(ctx, keys), dfree(ctx, ks), dfree(ctx, perm), dfree(ctx, hist), dfree(ctx, start);
                    throw;
                }
                dfree(ctx, keys), dfree(ctx, ks), dfree(ctx, perm), dfree(ctx, hist), dfree(ctx, start);
                release();
                return;
            }
            const u64 dn = span;  // dense bins over [0, span)
            dense = dalloc_t<unsigned long long>(ctx, dn);
            LO_CUDA(cudaMemsetAsync(dense, 0, 8 * dn, ctx->stream));
            const u64 e = res->rows * res->keff;
            if (e) {
                locality_dense<<<std::max(1, std::min(ceil_div(e, 256), ctx->sm_count * 4)), 256, 0,
                                 ctx->stream>>>(res->idx, res->rows, res->keff, cidx, map, dense);
                LO_CHECK_LAUNCH();
            }
            flags = dalloc_t<u32>(ctx, dn);
            pos = dalloc_t<u64>(ctx, dn + 1);
            const int g = std::max(1, std::min(ceil_div(dn, 256), ctx->sm_count * 16));
            nonzero_flags<<<g, 256, 0, ctx->stream>>>(dense, dn, flags);
            LO_CHECK_LAUNCH();
            exclusive_scan_u32_to_u64(ctx, flags, pos, dn);
            const u64 nb = read_scalar(ctx, pos + dn);
            *nbins = nb;
            if (d_host && count_host && nb <= cap && nb) {
                dd = dalloc_t<u32>(ctx, nb);
                cc = dalloc_t<u64>(ctx, nb);
                compact_bins<<<g, 256, 0, ctx->stream>>>(dense, pos, dn, dd, cc);
                LO_CHECK_LAUNCH();
                LO_CUDA(cudaMemcpyAsync(d_host, dd, 4 * nb, cudaMemcpyDeviceToHost, ctx->stream));
                LO_CUDA(cudaMemcpyAsync(count_host, cc, 8 * nb, cudaMemcpyDeviceToHost, ctx->stream));
            }
            sync(ctx);
        } catch (...) {
            release();
            throw;
        }
        release();
    });
}

}  // extern "C"
