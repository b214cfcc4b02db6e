// knn_float.cuh -- FP32-filtered exact kNN (K7), included by knn.cu.
//
// Exactness: the result is the first k points under (dist_sq, index) where dist_sq is the
// reference's FP64 point_dist_sq (search.cpp:180-185).  Each lane (query) keeps an FP64 max-heap
// of its k best; the FP32 copies only decide which candidates need the FP64 computation:
// with w = the heap's current worst dist_sq, a candidate (or a node's lower bound) whose FP32
// squared distance exceeds T(w) = w + M(w) provably has FP64 dist_sq > w, so it can neither
// enter the heap nor tie with its top (M(w) is the same error bound as the radius filter,
// evaluated at distance sqrt(w) with generous slack; search_common.cuh / DESIGN.md §4).
//
// Speed: for contiguous query ranges (Full mode) each tile first seeds its heaps from the
// contiguous SFC window around its 32 points -- spatially the nearest points -- so T is tight
// before the octree walk starts; the walk then enters a child only if some query's T reaches
// it, and candidates already seen in the window are skipped by index.
#pragma once

#include <type_traits>

#include "radius_float.cuh"

namespace lo {

struct KnnSmem {
    u32* stack;
    float* tq;      // per-query threshold T (FP32, +inf while the heap is not full)
    float4* qf;     // per-query FP32 coordinates
    float4* pa;     // staged candidate pairs (x0, x1, y0, y1)
    float2* pb;     // (z0, z1)
    u32* pidx;      // staged candidate indices
    u32* sidx;      // walk: leaf point indices gathered until 32 (then staged and offered together)
    double* pd;     // staged candidate FP64 coordinates (x, y, z per slot)
};

// Per-warp shared layout of knn_float_kernel (bytes): pd | stack | tq | qf | pa | pb | pidx
constexpr size_t kKnnOffPd = 0;
constexpr size_t kKnnOffStack = kKnnOffPd + 32 * 3 * 8;
constexpr size_t kKnnOffTq = kKnnOffStack + 4 * kStackCap;
constexpr size_t kKnnOffQf = kKnnOffTq + 4 * 32;
constexpr size_t kKnnOffPa = kKnnOffQf + 16 * 32;
constexpr size_t kKnnOffPb = kKnnOffPa + 16 * 16;
constexpr size_t kKnnOffPidx = kKnnOffPb + 8 * 16;
constexpr size_t kKnnOffSidx = kKnnOffPidx + 4 * 32;
constexpr size_t kKnnFixed = kKnnOffSidx + 4 * 32;

// T(w) = w + M(w) as an FP32 upper bound.  Evaluated in FP32 with every rounding directed up
// and a factor-3 slack on M (a larger T only admits more candidates to the exact FP64 test, so
// any overestimate is safe).
// The chain is evaluated with round-to-nearest FMAs and the hardware square-root approximation
// (sqrt.approx.f32, relative error <= 2^-23), each an upper bound after the final (1 + 2^-18)
// scaling: every term is non-negative, so the rounded sum is within 5 * 2^-24 of the directed-
// rounding one (the former __fsqrt_ru / __f*_ru chain cost ~8 % of the k = 16 kernel at cfg3).
__device__ __forceinline__ float knn_threshold(double w, float E) {
    const float u = 1.1920928955078125e-07f;  // 2^-23
    const float wf = __double2float_ru(w);
    float sw;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(sw) : "f"(wf));
    sw *= 1.0000038146972656f;  // 1 + 2^-18: an upper bound of sqrt(wf)
    const float dd = fmaf(2.0f * u, sw, 2.0f * E);
    float M = 12.0f * u * wf;
    M = fmaf(4.0f * 1.7320509f * sw, dd, M);
    M = fmaf(3.0f * dd, dd, M);
    M = fmaf(4.0e-15f, wf, M);
    return fmaf(3.0f, M, wf) * 1.0000038146972656f;
}

// The per-lane max-heap holds (key, index) with key = the FP64 dist_sq rounded up to FP32
// (8 bytes per entry instead of 12, so more warps fit in shared memory).  ru() is monotone, so
// different keys order exactly like the FP64 values; equal keys are resolved by recomputing both
// FP64 distances from the coordinates (the reference expression) and then the index.
__device__ __noinline__ bool key_tie_after(u32 ia, u32 ib, const double* __restrict__ px,
                                           const double* __restrict__ py, const double* __restrict__ pz,
                                           double cx, double cy, double cz) {
    if (ia == ib) return false;
    const double da = point_dist_sq(px[ia], py[ia], pz[ia], cx, cy, cz);
    const double db = point_dist_sq(px[ib], py[ib], pz[ib], cx, cy, cz);
    return da > db || (da == db && ia > ib);
}

struct KeyHeap {
    float* hk;
    u32* hi;
    u32 size;
    const double* __restrict__ px;
    const double* __restrict__ py;
    const double* __restrict__ pz;
    double cx, cy, cz;

    // (ka, ia) after (kb, ib) in (dist_sq, index) order; the rare equal-key case is out of line
    // so its coordinate loads are never hoisted into the common path
    __device__ __forceinline__ bool after(float ka, u32 ia, float kb, u32 ib) const {
        if (ka != kb) return ka > kb;
        return key_tie_after(ia, ib, px, py, pz, cx, cy, cz);
    }
    __device__ __forceinline__ void push(float k, u32 i) {
        u32 pos = size++;
        while (pos > 0) {
            const u32 par = (pos - 1) >> 1;
            const float pk = hk[par * 32];
            const u32 pi = hi[par * 32];
            if (!after(k, i, pk, pi)) break;
            hk[pos * 32] = pk;
            hi[pos * 32] = pi;
            pos = par;
        }
        hk[pos * 32] = k;
        hi[pos * 32] = i;
    }
    __device__ __forceinline__ void sift_down(float k, u32 i, u32 n) {
        u32 pos = 0;
        for (;;) {
            u32 c = 2 * pos + 1;
            if (c >= n) break;
            float ck = hk[c * 32];
            u32 ci = hi[c * 32];
            if (c + 1 < n) {
                const float rk = hk[(c + 1) * 32];
                const u32 ri = hi[(c + 1) * 32];
                if (after(rk, ri, ck, ci)) c = c + 1, ck = rk, ci = ri;
            }
            if (!after(ck, ci, k, i)) break;
            hk[pos * 32] = ck;
            hi[pos * 32] = ci;
            pos = c;
        }
        hk[pos * 32] = k;
        hi[pos * 32] = i;
    }
    template <int LOGK>
    __device__ __forceinline__ void sift_down_fixed(float k, u32 i) {
        constexpr u32 n = 1u << LOGK;
        u32 pos = 0;
#pragma unroll
        for (int lv = 0; lv < LOGK; ++lv) {
            u32 c = 2 * pos + 1;
            if (c >= n) break;
            float ck = hk[c * 32];
            u32 ci = hi[c * 32];
            if (c + 1 < n) {
                const float rk = hk[(c + 1) * 32];
                const u32 ri = hi[(c + 1) * 32];
                if (after(rk, ri, ck, ci)) c = c + 1, ck = rk, ci = ri;
            }
            if (!after(ck, ci, k, i)) break;
            hk[pos * 32] = ck;
            hi[pos * 32] = ci;
            pos = c;
        }
        hk[pos * 32] = k;
        hi[pos * 32] = i;
    }
};

// One candidate j (global index g, FP32 squared distance v) for this lane.
template <class Heap>
__device__ __forceinline__ Heap make_heap(typename std::conditional_t<std::is_same_v<Heap, KeyHeap>, float, double>* hd,
                                          u32* hi, const double* px, const double* py, const double* pz,
                                          double cx, double cy, double cz) {
    if constexpr (std::is_same_v<Heap, KeyHeap>) return KeyHeap{hd, hi, 0, px, py, pz, cx, cy, cz};
    else return LaneHeap{hd, hi, 0};
}

// Heap keys: LaneHeap keeps the exact FP64 dist_sq (12-byte entries), KeyHeap its FP32
// round-up (8-byte entries, more resident warps; chosen for k >= 32).
__device__ __forceinline__ double heap_key(const LaneHeap&, double d) { return d; }
__device__ __forceinline__ float heap_key(const KeyHeap&, double d) { return __double2float_ru(d); }
__device__ __forceinline__ double heap_root(const LaneHeap& h) { return h.hd[0]; }
__device__ __forceinline__ float heap_root(const KeyHeap& h) { return h.hk[0]; }

template <int KC, class Heap, class Key>
__device__ __forceinline__ void knn_offer(Heap& heap, u32 k, Key& worst_k, u32& worst_i,
                                          float& T, float E, float v, u32 g, double cx, double cy,
                                          double cz, const double* pxyz) {
    if (v > T) return;
    const double d = point_dist_sq(pxyz[0], pxyz[1], pxyz[2], cx, cy, cz);
    const Key kd = heap_key(heap, d);
    if (heap.size < k) {
        heap.push(kd, g);
        if (heap.size == k) {
            worst_k = heap_root(heap);
            worst_i = heap.hi[0];
            T = knn_threshold(static_cast<double>(worst_k), E);  // a key >= the exact worst: safe
        }
    } else if (heap.after(worst_k, worst_i, kd, g)) {
        if constexpr (KC == 8) heap.template sift_down_fixed<3>(kd, g);
        else if constexpr (KC == 16) heap.template sift_down_fixed<4>(kd, g);
        else if constexpr (KC == 32) heap.template sift_down_fixed<5>(kd, g);
        else if constexpr (KC == 64) heap.template sift_down_fixed<6>(kd, g);
        else heap.sift_down(kd, g, k);
        worst_k = heap_root(heap);
        worst_i = heap.hi[0];
        T = knn_threshold(static_cast<double>(worst_k), E);
    }
}

// Tests the `cnt` staged candidates against this lane's query (pairs, packed FP32).
template <int KC, class Heap, class Key>
__device__ __forceinline__ void knn_chunk_each(const KnnSmem& S, u32 cnt, bool active, u64 QX, u64 QY,
                                          u64 QZ, Heap& heap, u32 k, Key& worst_d,
                                          u32& worst_i, float& T, float E, double cx, double cy,
                                          double cz, u32 skip_lo, u32 skip_hi) {
    if (!active) return;
    const u32 npairs = (cnt + 1) >> 1;
    for (u32 pp = 0; pp < npairs; ++pp) {
        const float4 a = S.pa[pp];
        const float2 b = S.pb[pp];
        const u64 dx = fsub2(pack2(a.x, a.y), QX);
        const u64 dy = fsub2(pack2(a.z, a.w), QY);
        const u64 dz = fsub2(pack2(b.x, b.y), QZ);
        u64 d2 = fmul2(dx, dx);
        d2 = ffma2(dy, dy, d2);
        d2 = ffma2(dz, dz, d2);
        float v0, v1;
        unpack2(d2, v0, v1);
        if (v0 <= T) {
            const u32 g = S.pidx[2 * pp];
            if (g < skip_lo || g >= skip_hi)
                knn_offer<KC>(heap, k, worst_d, worst_i, T, E, v0, g, cx, cy, cz, S.pd + 6 * pp);
        }
        if (2 * pp + 1 < cnt && v1 <= T) {
            const u32 g = S.pidx[2 * pp + 1];
            if (g < skip_lo || g >= skip_hi)
                knn_offer<KC>(heap, k, worst_d, worst_i, T, E, v1, g, cx, cy, cz, S.pd + 6 * pp + 3);
        }
    }
}

// Tests the `cnt` staged candidates against this lane's query (pairs, packed FP32).  First every
// lane marks the candidates under its current threshold T, then the lanes offer their marked
// candidates in lockstep (ascending slot order, as before): once the heaps are full the passes are
// sparse and spread over the lanes, and offering candidate by candidate ran a warp-wide heap sift
// for every candidate any single lane wanted.  T only tightens, so re-checking a mark against the
// current T (knn_offer) keeps the result identical.  Measured faster for k = 8 only (6.98 vs 7.27 ms
// at cfg1); for k >= 16 the extra registers spill and it lost 3-7 %.
template <int KC, class Heap, class Key>
__device__ __forceinline__ void knn_chunk_marked(const KnnSmem& S, u32 cnt, bool active, u64 QX, u64 QY,
                                          u64 QZ, Heap& heap, u32 k, Key& worst_d,
                                          u32& worst_i, float& T, float E, double cx, double cy,
                                          double cz, u32 skip_lo, u32 skip_hi) {
    if (!active) return;
    const u32 npairs = (cnt + 1) >> 1;
    u32 pass = 0;
    for (u32 pp = 0; pp < npairs; ++pp) {
        const float4 a = S.pa[pp];
        const float2 b = S.pb[pp];
        const u64 dx = fsub2(pack2(a.x, a.y), QX);
        const u64 dy = fsub2(pack2(a.z, a.w), QY);
        const u64 dz = fsub2(pack2(b.x, b.y), QZ);
        u64 d2 = fmul2(dx, dx);
        d2 = ffma2(dy, dy, d2);
        d2 = ffma2(dz, dz, d2);
        float v0, v1;
        unpack2(d2, v0, v1);
        pass |= (v0 <= T ? 1u : 0u) << (2 * pp);
        pass |= (v1 <= T ? 1u : 0u) << (2 * pp + 1);
    }
    if (cnt < 32) pass &= (1u << cnt) - 1u;
    const float qx = __uint_as_float(static_cast<u32>(QX)), qy = __uint_as_float(static_cast<u32>(QY)),
                qz = __uint_as_float(static_cast<u32>(QZ));
    while (pass) {
        const int j = __ffs(pass) - 1;
        pass &= pass - 1;
        const u32 g = S.pidx[j];
        if (g >= skip_lo && g < skip_hi) continue;
        // the same FP32 expression as the packed one above (FADD2/FMUL2/FFMA2 are per-lane IEEE ops)
        const float* a = reinterpret_cast<const float*>(S.pa);
        const float* bb = reinterpret_cast<const float*>(S.pb);
        const int pp = j >> 1, h = j & 1;
        const float dx = a[4 * pp + h] - qx, dy = a[4 * pp + 2 + h] - qy, dz = bb[2 * pp + h] - qz;
        const float v = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
        knn_offer<KC>(heap, k, worst_d, worst_i, T, E, v, g, cx, cy, cz, S.pd + 3 * j);
    }
}

template <int KC, class Heap, class Key>
__device__ __forceinline__ void knn_chunk(const KnnSmem& S, u32 cnt, bool active, u64 QX, u64 QY,
                                          u64 QZ, Heap& heap, u32 k, Key& worst_d,
                                          u32& worst_i, float& T, float E, double cx, double cy,
                                          double cz, u32 skip_lo, u32 skip_hi) {
    if constexpr (KC == 8)
        knn_chunk_marked<KC>(S, cnt, active, QX, QY, QZ, heap, k, worst_d, worst_i, T, E, cx, cy, cz, skip_lo,
                             skip_hi);
    else
        knn_chunk_each<KC>(S, cnt, active, QX, QY, QZ, heap, k, worst_d, worst_i, T, E, cx, cy, cz, skip_lo,
                           skip_hi);
}

// Stage points [base, base + cnt) (cnt <= 32) of the sorted cloud: FP32 pairs for the filter,
// FP64 coordinates for the exact test of the candidates that pass it.
__device__ __forceinline__ void knn_stage(const KnnSmem& S, const float4* __restrict__ pf,
                                          const double* __restrict__ px, const double* __restrict__ py,
                                          const double* __restrict__ pz, u32 base, u32 cnt, int lane) {
    __syncwarp();
    if (static_cast<u32>(lane) < cnt) {
        const u32 g = base + lane;
        const float4 p = __ldg(pf + g);
        float* a = reinterpret_cast<float*>(S.pa);
        float* b = reinterpret_cast<float*>(S.pb);
        const int pp = lane >> 1, h = lane & 1;
        a[4 * pp + h] = p.x;
        a[4 * pp + 2 + h] = p.y;
        b[2 * pp + h] = p.z;
        S.pidx[lane] = g;
        S.pd[3 * lane] = __ldg(px + g);
        S.pd[3 * lane + 1] = __ldg(py + g);
        S.pd[3 * lane + 2] = __ldg(pz + g);
    }
    __syncwarp();
}

// Stage the `cnt` gathered candidates S.sidx[0, cnt) (any points of the sorted cloud).
__device__ __forceinline__ void knn_stage_idx(const KnnSmem& S, const float4* __restrict__ pf,
                                              const double* __restrict__ px, const double* __restrict__ py,
                                              const double* __restrict__ pz, u32 cnt, int lane) {
    __syncwarp();
    if (static_cast<u32>(lane) < cnt) {
        const u32 g = S.sidx[lane];
        const float4 p = __ldg(pf + g);
        float* a = reinterpret_cast<float*>(S.pa);
        float* b = reinterpret_cast<float*>(S.pb);
        const int pp = lane >> 1, h = lane & 1;
        a[4 * pp + h] = p.x;
        a[4 * pp + 2 + h] = p.y;
        b[2 * pp + h] = p.z;
        S.pidx[lane] = g;
        S.pd[3 * lane] = __ldg(px + g);
        S.pd[3 * lane + 1] = __ldg(py + g);
        S.pd[3 * lane + 2] = __ldg(pz + g);
    }
    __syncwarp();
}

#ifndef LO_KNN_PREFILTER_MIN_K
#define LO_KNN_PREFILTER_MIN_K 9
#endif
constexpr int kKnnFloatStack = kStackCap;
constexpr i64 kSeedSortedIdx = -2;  // seed_base: queries are ascending cloud indices (q.idx)

// -DLO_KNN_MINB=n sizes the register allocation for n resident blocks per SM (__launch_bounds__
// minimum); undefined leaves it to ptxas (80 registers at k = 16: 6 blocks of 4 warps per SM).
#ifdef LO_KNN_MINB
#define LO_KNN_BOUNDS __launch_bounds__(128, LO_KNN_MINB)
#else
#define LO_KNN_BOUNDS __launch_bounds__(128)
#endif
template <bool GLOBAL_HEAP, int KC, bool KEYED>
__global__ void LO_KNN_BOUNDS knn_float_kernel(
    const TNodeF* __restrict__ tf, const float4* __restrict__ pf, const double* __restrict__ px,
    const double* __restrict__ py, const double* __restrict__ pz, u64 npoints, Queries q,
    i64 seed_base, u32 seed_half, float E, u32 k_in, u32* __restrict__ out_idx,
    double* __restrict__ out_dist, void* __restrict__ gheap_d, u32* __restrict__ gheap_i,
    u64* tile_counter) {
    extern __shared__ __align__(16) unsigned char smem[];
    using Heap = std::conditional_t<KEYED, KeyHeap, LaneHeap>;
    using Key = std::conditional_t<KEYED, float, double>;
    const u32 k = KC > 0 ? static_cast<u32>(KC) : k_in;
    const int warps = blockDim.x >> 5;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned char* mine = smem + w * kKnnFixed;
    KnnSmem S;
    S.pd = reinterpret_cast<double*>(mine + kKnnOffPd);
    S.stack = reinterpret_cast<u32*>(mine + kKnnOffStack);
    S.tq = reinterpret_cast<float*>(mine + kKnnOffTq);
    S.qf = reinterpret_cast<float4*>(mine + kKnnOffQf);
    S.pa = reinterpret_cast<float4*>(mine + kKnnOffPa);
    S.pb = reinterpret_cast<float2*>(mine + kKnnOffPb);
    S.pidx = reinterpret_cast<u32*>(mine + kKnnOffPidx);
    S.sidx = reinterpret_cast<u32*>(mine + kKnnOffSidx);
    Key* hd;
    u32* hi;
    if (GLOBAL_HEAP) {
        const u64 slot = static_cast<u64>(blockIdx.x) * warps + w;
        hd = static_cast<Key*>(gheap_d) + slot * k * 32 + lane;
        hi = gheap_i + slot * k * 32 + lane;
    } else {
        Key* heaps_d = reinterpret_cast<Key*>(smem + warps * kKnnFixed);
        u32* heaps_i = reinterpret_cast<u32*>(heaps_d + static_cast<u64>(warps) * k * 32);
        hd = heaps_d + static_cast<u64>(w) * k * 32 + lane;
        hi = heaps_i + static_cast<u64>(w) * k * 32 + lane;
    }
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
        const u64 QX = pack2(qf.x, qf.x), QY = pack2(qf.y, qf.y), QZ = pack2(qf.z, qf.z);
        Heap heap = make_heap<Heap>(hd, hi, px, py, pz, cx, cy, cz);
        Key worst_d = 0;
        u32 worst_i = 0;
        float T = active ? INFINITY : -INFINITY;  // inactive lanes want nothing
        __syncwarp();
        S.qf[lane] = qf;

        // 1) seed from the contiguous SFC window around the tile (Full / range mode)
        u32 skip_lo = 0, skip_hi = 0;
        i64 t0 = 0, t1 = -1;
        if (seed_base >= 0) {
            t0 = seed_base + static_cast<i64>(tile * 32);
            t1 = seed_base + static_cast<i64>(min(q.m, tile * 32 + 32));
        } else if (seed_base == kSeedSortedIdx) {
            // ascending centre indices: seed from their window when the tile is dense along the
            // curve; a sparse tile (random subset) seeds every lane from its own centre's window
            t0 = q.idx[tile * 32];
            t1 = static_cast<i64>(q.idx[min(q.m, tile * 32 + 32) - 1]) + 1;
            if (t1 - t0 > 4 * 32 || t1 <= t0) {  // spread out (or unsorted: caller's order)
                t1 = -1;
                if (active) {
                    const i64 c = q.idx[qi];
                    i64 lo = c - static_cast<i64>(seed_half / 2);
                    if (lo < 0) lo = 0;
                    i64 hi_ = lo + static_cast<i64>(seed_half);
                    if (hi_ > static_cast<i64>(npoints)) {
                        hi_ = static_cast<i64>(npoints);
                        lo = hi_ - static_cast<i64>(seed_half) < 0 ? 0 : hi_ - static_cast<i64>(seed_half);
                    }
                    skip_lo = static_cast<u32>(lo);
                    skip_hi = static_cast<u32>(hi_);
                    for (u32 g = skip_lo; g < skip_hi; ++g) {
                        const float4 p = __ldg(pf + g);
                        const float dx = p.x - qf.x, dy = p.y - qf.y, dz = p.z - qf.z;
                        const float v = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
                        if (v <= T) {
                            const double pd[3] = {__ldg(px + g), __ldg(py + g), __ldg(pz + g)};
                            knn_offer<KC>(heap, k, worst_d, worst_i, T, E, v, g, cx, cy, cz, pd);
                        }
                    }
                }
            }
        }
        if (t1 >= 0) {
            i64 lo = t0 - static_cast<i64>(seed_half);
            if (lo < 0) lo = 0;
            i64 hi_ = t1 + static_cast<i64>(seed_half);
            if (hi_ > static_cast<i64>(npoints)) hi_ = static_cast<i64>(npoints);
            skip_lo = static_cast<u32>(lo);
            skip_hi = static_cast<u32>(hi_);
            for (u32 b = skip_lo; b < skip_hi; b += 32) {
                const u32 cnt = min(32u, skip_hi - b);
                knn_stage(S, pf, px, py, pz, b, cnt, lane);
                knn_chunk<KC>(S, cnt, active, QX, QY, QZ, heap, k, worst_d, worst_i, T, E, cx, cy, cz,
                          0u, 0u);
            }
        }

        // 2) octree walk; a node is entered if some query's threshold reaches its box
        u32 kfill = 0;
        bool kwant = false;
        // Point prefilter for the gathered leaves (as in the radius walk; k >= 16 -- k = 8's thresholds
        // are tight enough that the filter costs more, 6.77 -> 7.07 ms at cfg1; k = 16: cfg3 149.7 ->
        // 144.5 ms, cfg1 11.93 -> 11.82 ms): a candidate whose FP32 squared distance to the tile's
        // query box exceeds every lane's threshold T would be rejected by every lane (each lane's
        // d2 >= the box value: per axis |p - q| >= the gap and the FP32 ops are monotone), so it is
        // dropped before it takes a slot.  max_t is a stale upper bound of the lanes' T (T only
        // decreases), refreshed after each flush.
        constexpr bool KPF = !KEYED && KC >= LO_KNN_PREFILTER_MIN_K;
        float tb[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        auto warp_max_t = [&]() {
            float m = T;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(~0u, m, o));
            return m;
        };
        float max_t = INFINITY;
        if constexpr (KPF) {
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const float c = a == 0 ? qf.x : (a == 1 ? qf.y : qf.z);
                float lo_ = c, hi_ = c;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    lo_ = fminf(lo_, __shfl_xor_sync(~0u, lo_, o));
                    hi_ = fmaxf(hi_, __shfl_xor_sync(~0u, hi_, o));
                }
                tb[a] = lo_, tb[3 + a] = hi_;
            }
            max_t = warp_max_t();
        }
        auto kflush = [&]() {
            knn_stage_idx(S, pf, px, py, pz, kfill, lane);
            knn_chunk<KC>(S, kfill, kwant, QX, QY, QZ, heap, k, worst_d, worst_i, T, E, cx, cy, cz, skip_lo,
                          skip_hi);
            kfill = 0;
            kwant = false;
            if constexpr (KPF) max_t = warp_max_t();
        };
        int sp = 1;
        if (lane == 0) S.stack[0] = 0;
        __syncwarp();
        while (sp > 0) {
            __syncwarp();
            S.tq[lane] = T;
            __syncwarp();
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
                        keep |= fmaf(nz, nz, fmaf(ny, ny, nx * nx)) <= S.tq[8 * grp + j];
                    }
                }
                u32 s = __ballot_sync(~0u, keep);
                s = (s | (s >> 8) | (s >> 16) | (s >> 24)) & 0xffu;
                const int kk = __popc(s);
                __syncwarp();
                if (lane < 8 && ((s >> lane) & 1u))
                    S.stack[sp + kk - 1 - __popc(s & ((1u << lane) - 1u))] = nd.child0 + lane;
                sp += kk;
                continue;
            }
            // leaf: skip if no lane's threshold reaches it, or it lies inside the seed window
            if (__all_sync(~0u, nd.begin >= skip_lo && nd.end <= skip_hi)) continue;  // seeded already
            bool want = false;
            if (active) {
                const float nx = fmaxf(fmaxf(nd.lo[0] - qf.x, qf.x - nd.hi[0]), 0.f);
                const float ny = fmaxf(fmaxf(nd.lo[1] - qf.y, qf.y - nd.hi[1]), 0.f);
                const float nz = fmaxf(fmaxf(nd.lo[2] - qf.z, qf.z - nd.hi[2]), 0.f);
                want = fmaf(nz, nz, fmaf(ny, ny, nx * nx)) <= T;
            }
            if (!__any_sync(~0u, want)) continue;
            if constexpr (KEYED) {  // k >= 32: per leaf (gathering spilled and loosened T: +21-35 %)
                for (u32 b = nd.begin; b < nd.end; b += 32) {
                    const u32 cnt = min(32u, nd.end - b);
                    knn_stage(S, pf, px, py, pz, b, cnt, lane);
                    knn_chunk<KC>(S, cnt, want, QX, QY, QZ, heap, k, worst_d, worst_i, T, E, cx, cy, cz,
                                  skip_lo, skip_hi);
                }
            } else {
                // gather the leaf's indices; 32 of them (from several small leaves) are staged and
                // offered at once -- one load latency per 32 candidates instead of one per leaf
                // (k = 8: 6.98 -> 6.55 ms, k = 16: 11.17 -> 11.03 ms at cfg1)
                if constexpr (KPF) {
                for (u32 b0 = nd.begin; b0 < nd.end; b0 += 32) {
                    const u32 g = b0 + static_cast<u32>(lane);
                    bool ok = false;
                    if (g < nd.end) {
                        const float4 pp = __ldg(pf + g);
                        const float gx = fmaxf(fmaxf(tb[0] - pp.x, pp.x - tb[3]), 0.f);
                        const float gy = fmaxf(fmaxf(tb[1] - pp.y, pp.y - tb[4]), 0.f);
                        const float gz = fmaxf(fmaxf(tb[2] - pp.z, pp.z - tb[5]), 0.f);
                        ok = __fmaf_rn(gz, gz, __fmaf_rn(gy, gy, __fmul_rn(gx, gx))) <= max_t;
                    }
                    const u32 bal = __ballot_sync(~0u, ok);
                    if (!bal) continue;
                    const u32 pos = kfill + __popc(bal & ((1u << lane) - 1u));
                    __syncwarp();
                    if (ok && pos < 32) S.sidx[pos] = g;
                    kfill += __popc(bal);
                    kwant |= want;
                    if (kfill >= 32) {
                        const u32 over = kfill - 32;
                        kfill = 32;
                        __syncwarp();
                        kflush();
                        __syncwarp();
                        if (ok && pos >= 32) S.sidx[pos - 32] = g;
                        kfill = over;
                        kwant = over ? want : false;
                    }
                }
                } else {
                for (u32 b = nd.begin; b < nd.end;) {
                    const u32 take = min(32u - kfill, nd.end - b);
                    __syncwarp();
                    if (static_cast<u32>(lane) < take) S.sidx[kfill + lane] = b + lane;
                    kfill += take;
                    kwant |= want;
                    b += take;
                    if (kfill == 32) kflush();
                }
                }
            }
        }
        if (kfill) kflush();

        // 3) heap sort in place -> ascending (dist_sq, index); coalesced row writes
        if (active) {
            const u32 n = heap.size;
            for (u32 e = n; e > 1; --e) {
                const Key td = hd[0];
                const u32 ti = hi[0];
                const Key ld = hd[(e - 1) * 32];
                const u32 li = hi[(e - 1) * 32];
                hd[(e - 1) * 32] = td;
                hi[(e - 1) * 32] = ti;
                heap.sift_down(ld, li, e - 1);
            }
        }
        __syncwarp();
        const u64 left = q.m - tile * 32;
        const u32 nact = left < 32 ? static_cast<u32>(left) : 32u;
        for (u32 L = 0; L < nact; ++L) {
            // the row's FP64 distances are recomputed with the reference expression
            const double qx = __shfl_sync(~0u, cx, L), qy = __shfl_sync(~0u, cy, L), qz = __shfl_sync(~0u, cz, L);
            u32* oi = out_idx + (tile * 32 + L) * k;
            double* od = out_dist + (tile * 32 + L) * k;
            const u32* rhi = hi - lane + L;
            const Key* rhd = hd - lane + L;
            for (u32 e = lane; e < k; e += 32) {
                const u32 j = rhi[e * 32];
                oi[e] = j;
                if constexpr (KEYED)
                    od[e] = point_dist_sq(__ldg(px + j), __ldg(py + j), __ldg(pz + j), qx, qy, qz);
                else
                    od[e] = rhd[e * 32];
            }
        }
        __syncwarp();
    }
}

}  // namespace lo
