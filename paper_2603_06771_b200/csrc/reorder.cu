// reorder.cu -- K1 bbox, K2 encode (+ fused digit histograms), K3 onesweep LSD radix sort,
// K4 SoA gather.  Replaces compute_codes / radix_sort_codes / reorder_cloud
// (reorder.cpp:9-89) with bit-identical results (keys, stable permutation, coordinates).
#include <cstring>
#include <cub/block/block_scan.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>

#include "lo_internal.cuh"

namespace lo {

// ---- K1: exact bbox + finite check (geometry.hpp:64-82) ----------------------------------
// min/max are taken on the order-preserving integer image, so the reduction is exact and
// order independent.  bbox[0..2] = min keys, [3..5] = max keys, [6] = first non-finite index.
__global__ void __launch_bounds__(256) bbox_kernel(const double* __restrict__ xyz, u64 n,
                                                   u64* __restrict__ out) {
    u64 mn[3] = {~0ull, ~0ull, ~0ull}, mx[3] = {0, 0, 0};
    u64 bad = ~0ull;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n;
         i += (u64)gridDim.x * blockDim.x) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double v = xyz[3 * i + a];
            if (!isfinite(v)) bad = min(bad, i);
            const u64 k = dbl_order_key(v);
            mn[a] = min(mn[a], k);
            mx[a] = max(mx[a], k);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            mn[a] = min(mn[a], __shfl_xor_sync(~0u, mn[a], o));
            mx[a] = max(mx[a], __shfl_xor_sync(~0u, mx[a], o));
        }
        bad = min(bad, __shfl_xor_sync(~0u, bad, o));
    }
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            atomicMin(reinterpret_cast<unsigned long long*>(out + a), mn[a]);
            atomicMax(reinterpret_cast<unsigned long long*>(out + 3 + a), mx[a]);
        }
        if (bad != ~0ull) atomicMin(reinterpret_cast<unsigned long long*>(out + 6), bad);
    }
}

__global__ void bbox_init(u64* out) {
    const int t = threadIdx.x;
    if (t < 3) out[t] = ~0ull;
    else if (t < 6) out[t] = 0;
    else if (t == 6) out[t] = ~0ull;
}

// ---- K2: quantise + encode, with the 8 byte-digit histograms of the sort fused in --------
struct EncodeParams {
    double lo[3];
    double hi[3];     // closed-box check (sfc.hpp:105)
    double scale[3];
    double top;       // 2^level - 1 as double (sfc.hpp:122)
    int level;
    int curve;
    u8 enc[32 * 8];   // Hilbert / Morton encode table (state, octant) -> digit | next << 3
    const u16* h3;    // Hilbert: three levels per step, (state, 9 Morton bits) -> 9 code bits | next << 9
};

constexpr int kH3States = 24;
constexpr int kH3Entries = kH3States * 512;

// axis_cell (sfc.hpp:120-124): floor((v - lo) * scale), clamped to [0, top].
__device__ __forceinline__ u32 axis_cell(double v, double lo, double scale, double top) {
    double u = floor((v - lo) * scale);
    u = u < 0.0 ? 0.0 : (top < u ? top : u);
    return static_cast<u32>(u);
}

__device__ __forceinline__ u64 encode_cell(u32 cx, u32 cy, u32 cz, int level, int curve,
                                           const u8* enc, const u16* h3) {
    // the Morton code's 3-bit digits are the octant digits g = x<<2 | y<<1 | z of every level
    const u64 m = (spread3(cx) << 2) | (spread3(cy) << 1) | spread3(cz);
    if (curve == LO_MORTON) return m;
    // Hilbert: walk the 24-state descent table from the root (equivalent to the Skilling
    // transform of sfc.cpp:8-42; pinned by tests against the reference) -- level % 3 single
    // levels, then three levels (9 Morton bits) per table step: 7 dependent lookups at level 21
    // instead of 21.
    u64 code = 0;
    u32 s = 0;
    int d = level - 1;
    for (; (d + 1) % 3 != 0; --d) {
        const u32 e = enc[s * 8 + ((m >> (3 * d)) & 7u)];
        code = (code << 3) | (e & 7u);
        s = e >> 3;
    }
    for (d -= 2; d >= 0; d -= 3) {
        const u32 e = h3[s * 512 + ((m >> (3 * d)) & 511u)];
        code = (code << 9) | (e & 511u);
        s = e >> 9;
    }
    return code;
}

// Shared-memory copy of the three-level Hilbert table (Morton never reads it).
__device__ __forceinline__ void load_h3(u16* dst, const EncodeParams& p) {
    if (p.curve != LO_HILBERT) return;
    const uint4* src = reinterpret_cast<const uint4*>(p.h3);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (int i = threadIdx.x; i < kH3Entries * 2 / 16; i += blockDim.x) d4[i] = src[i];
}

template <bool HIST>
__global__ void __launch_bounds__(256) encode_kernel(const double* __restrict__ xyz, u64 n,
                                                     EncodeParams p, u64* __restrict__ codes,
                                                     u32* __restrict__ hist, u32* __restrict__ err) {
    __shared__ u8 enc[32 * 8];
    __shared__ __align__(16) u16 h3[kH3Entries];
    __shared__ u32 h[HIST ? 8 * 256 : 1];
    for (int i = threadIdx.x; i < 32 * 8; i += blockDim.x) enc[i] = p.enc[i];
    load_h3(h3, p);
    if (HIST)
        for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) h[i] = 0;
    __syncthreads();
    u32 outside = 0;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n;
         i += (u64)gridDim.x * blockDim.x) {
        const double x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
        if (!(x >= p.lo[0] && x <= p.hi[0] && y >= p.lo[1] && y <= p.hi[1] && z >= p.lo[2] &&
              z <= p.hi[2]))
            outside = 1;
        const u32 cx = axis_cell(x, p.lo[0], p.scale[0], p.top);
        const u32 cy = axis_cell(y, p.lo[1], p.scale[1], p.top);
        const u32 cz = axis_cell(z, p.lo[2], p.scale[2], p.top);
        const u64 code = encode_cell(cx, cy, cz, p.level, p.curve, enc, h3);
        codes[i] = code;
        if (HIST) {
#pragma unroll
            for (int b = 0; b < 8; ++b) atomicAdd(&h[b * 256 + ((code >> (8 * b)) & 0xff)], 1u);
        }
    }
    if (outside) atomicOr(err, 1u);
    if (HIST) {
        __syncthreads();
        for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x)
            if (h[i]) atomicAdd(&hist[i], h[i]);
    }
}

// ---- K3: onesweep LSD radix sort pass (8-bit digit, stable, decoupled look-back) ---------
// Tile = 256 threads x kSortItems keys; warp w owns keys [w*32*I, (w+1)*32*I) in (item, lane)
// order.  Each warp ranks its keys with __match_any_sync; the per-item running counts go through
// one shared-memory atomic per distinct digit, issued back to back (a warp's shared atomics
// execute in program order, so equal digits keep input order) instead of a load / store /
// __syncwarp chain per item.  Tiles chain their per-digit totals through a look-back status word
// per (tile, digit): flag (2 bits) | pass epoch (6 bits) | count (56 bits), so one memset per sort
// serves every pass.  Order inside a tile: (1) ranking, (2) local offsets and the tile's
// aggregate published, (3) the tile is scattered into shared memory and its values loaded,
// (4) only then the look-back for the global digit prefix (predecessors had the scatter's time to
// publish), (5) coalesced global writes.  The look-back reads LO_SORT_LB = 4 predecessors per
// L2 round trip.  cfg3 sort 9.04 -> 6.62 ms, cfg1 1.124 -> 0.966 ms (torch.sort / CUB SortPairs
// on the same counts of 64-bit keys: 8.61 / 1.03 ms; profiles/r2b/sort_v2.log, sort_lookback.log;
// one predecessor per round trip: 7.77 / 1.046 ms, eight: 6.66 / 0.974 ms).  LO_SORT_EARLY=1 publishes an early block histogram (shared
// atomics) before the ranking instead; measured slower (8.09 / 1.073 ms).
constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
#ifndef LO_SORT_ITEMS
#define LO_SORT_ITEMS 12
#endif
#ifndef LO_SORT_MINB
#define LO_SORT_MINB 4
#endif
#ifndef LO_SORT_EARLY
#define LO_SORT_EARLY 0
#endif
#ifndef LO_SORT_GROUP
#define LO_SORT_GROUP 4
#endif
#ifndef LO_SORT_LB
#define LO_SORT_LB 4
#endif
constexpr int kSortItems = LO_SORT_ITEMS;
constexpr int kSortTile = kSortThreads * kSortItems;
constexpr u64 kFlagAgg = 1ull << 62, kFlagInc = 2ull << 62, kFlagMask = 3ull << 62;
constexpr int kEpochShift = 56;
constexpr u64 kCountMask = (1ull << kEpochShift) - 1;

struct SortSmem {
    u64 keys[kSortTile];
    u32 vals[kSortTile];
    u32 whist[kSortWarps][256];
    u32 local_start[256];
    u32 bhist[256];
    u64 gofs[256];
    u32 tile;
    typename cub::BlockScan<u32, kSortThreads>::TempStorage scan;
};

template <bool FIRST>
__global__ void __launch_bounds__(kSortThreads, LO_SORT_MINB) onesweep_pass(
    const u64* __restrict__ kin, const u32* __restrict__ vin, u64* __restrict__ kout,
    u32* __restrict__ vout, u64 n, int shift, const u64* __restrict__ digit_base,
    u64* status_, u32* counter, u32 epoch) {
    volatile u64* status = status_;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SortSmem& S = *reinterpret_cast<SortSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (tid == 0) S.tile = atomicAdd(counter, 1u);
    for (int i = tid; i < kSortWarps * 256; i += kSortThreads) (&S.whist[0][0])[i] = 0;
    if (LO_SORT_EARLY) S.bhist[tid] = 0;
    __syncthreads();
    const u32 tile = S.tile;
    const u64 base = static_cast<u64>(tile) * kSortTile;
    const u64 wbase = base + static_cast<u64>(w) * (32 * kSortItems);
    const u64 ep = static_cast<u64>(epoch) << kEpochShift;
    volatile u64* st = status + static_cast<u64>(tile) * 256;

    u64 key[kSortItems];
    u32 rank[kSortItems];
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
        const u64 idx = wbase + i * 32 + lane;
        key[i] = idx < n ? kin[idx] : ~0ull;  // pad keys: digit 255, ranked last
    }
    const u64 tile_n = min(static_cast<u64>(kSortTile), n - base);
    if (LO_SORT_EARLY) {
        // early block histogram, so successors see this tile's aggregate while it ranks
#pragma unroll
        for (int i = 0; i < kSortItems; ++i)
            if (wbase + i * 32 + lane < n) atomicAdd(&S.bhist[(key[i] >> shift) & 0xff], 1u);
        __syncthreads();
        st[tid] = (tile == 0 ? kFlagInc : kFlagAgg) | ep | S.bhist[tid];
    }
    // (1) ranking: match a group of items, then one leader atomic per distinct digit and item
    constexpr int G = LO_SORT_GROUP;
    static_assert(kSortItems % G == 0, "items per thread must be a multiple of the match group");
    const u32 lt = (1u << lane) - 1u;
#pragma unroll
    for (int i0 = 0; i0 < kSortItems; i0 += G) {
        u32 peers[G], old[G];
#pragma unroll
        for (int u = 0; u < G; ++u) {
            const u32 d = static_cast<u32>((key[i0 + u] >> shift) & 0xff);
            peers[u] = __match_any_sync(~0u, d);
        }
#pragma unroll
        for (int u = 0; u < G; ++u) {
            const u32 d = static_cast<u32>((key[i0 + u] >> shift) & 0xff);
            old[u] = 0;
            if (lane == __ffs(peers[u]) - 1) old[u] = atomicAdd(&S.whist[w][d], static_cast<u32>(__popc(peers[u])));
        }
#pragma unroll
        for (int u = 0; u < G; ++u)
            rank[i0 + u] = __shfl_sync(~0u, old[u], __ffs(peers[u]) - 1) + __popc(peers[u] & lt);
    }
    __syncthreads();

    // (2) per digit: exclusive offsets across warps, tile total, local starts
    const int d = tid;
    u32 total = 0;
#pragma unroll
    for (int ww = 0; ww < kSortWarps; ++ww) {
        const u32 c = S.whist[ww][d];
        S.whist[ww][d] = total;
        total += c;
    }
    // pad keys sit at the top of digit 255: drop them from the published count
    const u32 pad = static_cast<u32>(kSortTile - tile_n);
    const u32 real = d == 255 ? total - pad : total;
    if (!LO_SORT_EARLY) st[d] = (tile == 0 ? kFlagInc : kFlagAgg) | ep | real;
    u32 lstart;
    cub::BlockScan<u32, kSortThreads>(S.scan).ExclusiveSum(total, lstart);
    S.local_start[d] = lstart;
    __syncthreads();

    // (3) scatter the tile into shared memory in digit order; load the values meanwhile
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
        const u32 dd = static_cast<u32>((key[i] >> shift) & 0xff);
        const u32 pos = S.local_start[dd] + S.whist[w][dd] + rank[i];
        S.keys[pos] = key[i];
        rank[i] = pos;
    }
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
        const u64 idx = wbase + i * 32 + lane;
        const u32 v = FIRST ? static_cast<u32>(idx) : (idx < n ? vin[idx] : 0u);
        S.vals[rank[i]] = v;
    }

    // (4) look back for this digit's global prefix, LO_SORT_LB predecessors per round trip (the
    // walk over predecessors that only published their aggregate is a chain of L2 round trips)
    u64 excl = 0;
    if (tile > 0) {
        constexpr int W = LO_SORT_LB;
        i64 j = static_cast<i64>(tile) - 1;
        bool done = false;
        while (!done) {
            u64 s[W];
#pragma unroll
            for (int u = 0; u < W; ++u)
                s[u] = j - u >= 0 ? status[static_cast<u64>(j - u) * 256 + d] : (kFlagInc | ep);
            // status words are read with ld.volatile (above: `status` is accessed through a
            // volatile pointer); consume them nearest first, retry from the first empty one
            int u = 0;
            for (; u < W; ++u) {
                const u64 f = s[u] & kFlagMask;
                if (f == 0 || (s[u] & ~kFlagMask) >> kEpochShift != epoch) break;
                excl += s[u] & kCountMask;
                if (f == kFlagInc) {
                    done = true;
                    break;
                }
            }
            if (!done) j -= u;
        }
        st[d] = kFlagInc | ep | (excl + real);
    }
    S.gofs[d] = digit_base[d] + excl - lstart;
    __syncthreads();

    // (5) coalesced global writes: consecutive threads write consecutive slots of a digit run
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
        const u32 p = i * kSortThreads + tid;
        if (p < tile_n) {
            const u64 k = S.keys[p];
            const u64 gp = S.gofs[(k >> shift) & 0xff] + p;
            kout[gp] = k;
            vout[gp] = S.vals[p];
        }
    }
}

// ---- K4: gather into SFC order, SoA f64 ---------------------------------------------------
// Also writes the FP32 filter copy fl32(fl64(p - origin)) (search_common.cuh error bounds).
#ifndef LO_GATHER_ILP
#define LO_GATHER_ILP 4
#endif
// The scattered 24-byte record reads of the gather, with the L2 fetch size cut to 64 bytes: the
// default fetched 128 per miss, ~145 B of DRAM reads per record (cfg3 gather: 14.5 -> 8.3 GB of
// DRAM reads, 3.45 -> 3.38 ms).  The L1 keeps allocating: x, y, z of a record share its sector
// (L1::no_allocate measured 6.4 ms).  LO_GATHER_PLAIN=1: plain loads.
__device__ __forceinline__ double gather_ld(const double* p) {
#if LO_GATHER_PLAIN
    return *p;
#else
    double v;
    asm volatile("ld.global.nc.L2::64B.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
#endif
}
// Each thread keeps LO_GATHER_ILP random record gathers in flight (the perm loads first, then all
// coordinate loads, then the stores): the source records are scattered 24-byte reads.
__global__ void __launch_bounds__(256) gather_soa(const double* __restrict__ xyz,
                                                  const u32* __restrict__ perm, u64 n,
                                                  double* __restrict__ x, double* __restrict__ y,
                                                  double* __restrict__ z, float4* __restrict__ pf,
                                                  double ox, double oy, double oz) {
    constexpr int U = LO_GATHER_ILP;
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 i0 = blockIdx.x * (u64)blockDim.x + threadIdx.x; i0 < n; i0 += U * stride) {
        u64 o[U];
        double a[U], b[U], c[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const u64 i = i0 + u * stride;
            o[u] = i < n ? perm[i] : 0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (i0 + u * stride < n) {
                a[u] = gather_ld(xyz + 3 * o[u]);
                b[u] = gather_ld(xyz + 3 * o[u] + 1);
                c[u] = gather_ld(xyz + 3 * o[u] + 2);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const u64 i = i0 + u * stride;
            if (i < n) {
                x[i] = a[u];
                y[i] = b[u];
                z[i] = c[u];
                pf[i] = make_float4(__double2float_rn(a[u] - ox), __double2float_rn(b[u] - oy),
                                    __double2float_rn(c[u] - oz), 0.f);
            }
        }
    }
}

__global__ void __launch_bounds__(256) float_points(const double* __restrict__ x,
                                                    const double* __restrict__ y,
                                                    const double* __restrict__ z, u64 n,
                                                    float4* __restrict__ pf, double ox, double oy,
                                                    double oz) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n;
         i += (u64)gridDim.x * blockDim.x)
        pf[i] = make_float4(__double2float_rn(x[i] - ox), __double2float_rn(y[i] - oy),
                            __double2float_rn(z[i] - oz), 0.f);
}

void build_float_points(lo_context* ctx, lo_coded* c) {
    if (c->pf) return;
    c->pf = dalloc_t<float4>(ctx, c->n);
    float_points<<<std::max<u64>(1, std::min<u64>((c->n + 255) / 256, ctx->sm_count * 8ull)), 256, 0,
                   ctx->stream>>>(c->x, c->y, c->z, c->n, c->pf, c->origin[0], c->origin[1],
                                  c->origin[2]);
    LO_CHECK_LAUNCH();
}

static void set_origin(lo_coded* c) {
    for (int a = 0; a < 3; ++a) c->origin[a] = c->disc_box[a];
    c->bmax = std::max({c->disc_box[3] - c->disc_box[0], c->disc_box[4] - c->disc_box[1],
                        c->disc_box[5] - c->disc_box[2]});
}

__global__ void iota_u32(u32* p, u64 n) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n;
         i += (u64)gridDim.x * blockDim.x)
        p[i] = static_cast<u32>(i);
}

__global__ void interleave_aos(const double* __restrict__ x, const double* __restrict__ y,
                               const double* __restrict__ z, u64 n, double* __restrict__ xyz) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n;
         i += (u64)gridDim.x * blockDim.x) {
        xyz[3 * i] = x[i];
        xyz[3 * i + 1] = y[i];
        xyz[3 * i + 2] = z[i];
    }
}

__global__ void invert_perm_kernel(const u32* __restrict__ perm, u64 n, u32* __restrict__ inv) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n;
         i += (u64)gridDim.x * blockDim.x)
        inv[perm[i]] = static_cast<u32>(i);
}

__global__ void encode_cells_kernel(const u32* __restrict__ cells, u64 n, int level, int curve,
                                    EncodeParams p, u64* __restrict__ codes) {
    __shared__ u8 enc[32 * 8];
    __shared__ __align__(16) u16 h3[kH3Entries];
    for (int i = threadIdx.x; i < 32 * 8; i += blockDim.x) enc[i] = p.enc[i];
    load_h3(h3, p);
    __syncthreads();
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n;
         i += (u64)gridDim.x * blockDim.x)
        codes[i] = encode_cell(cells[3 * i], cells[3 * i + 1], cells[3 * i + 2], level, curve, enc, h3);
}

__global__ void decode_codes_kernel(const u64* __restrict__ codes, u64 n, int level,
                                    const CurveTables tab, u32* __restrict__ cells) {
    __shared__ u8 dec[32 * 8];
    for (int i = threadIdx.x; i < 32 * 8; i += blockDim.x) dec[i] = tab.dec[i];
    __syncthreads();
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n;
         i += (u64)gridDim.x * blockDim.x) {
        const u64 c = codes[i];
        u32 x = 0, y = 0, z = 0, s = 0;
        for (int d = level - 1; d >= 0; --d) {
            const u32 e = dec[s * 8 + ((c >> (3 * d)) & 7u)];
            x = x << 1 | ((e >> 2) & 1u);
            y = y << 1 | ((e >> 1) & 1u);
            z = z << 1 | (e & 1u);
            s = e >> 3;
        }
        cells[3 * i] = x, cells[3 * i + 1] = y, cells[3 * i + 2] = z;
    }
}

// encode blocks per SM (A/B knob LO_ENCODE_PER_SM; 33 KB of shared memory each, at most 6 resident;
// 8 measured best: cfg3 encode 1.21 / 1.19 / 1.16 / 1.11 ms at 4 / 5 / 6 / 8, profiles/r3/encode_ab.log)
static int encode_per_sm() {
    static const int v = [] {
        const char* e = std::getenv("LO_ENCODE_PER_SM");
        return e ? std::max(1, std::atoi(e)) : 8;
    }();
    return v;
}
static int grid_for(lo_context* ctx, u64 n, int threads, int per_sm = 8) {
    const u64 want = (n + threads - 1) / threads;
    const u64 cap = static_cast<u64>(ctx->sm_count) * per_sm;
    return static_cast<int>(std::max<u64>(1, std::min(want, cap)));
}

// ---- host: bbox -> Discretizer (cubify, axis_scale) exactly as the reference ------------
struct Disc {
    double cloud_box[6];
    double box[6];
    double scale[3];
};

static Disc compute_disc(lo_context* ctx, const double* xyz_dev, u64 n, int level) {
    u64* bb = dalloc_t<u64>(ctx, 8);
    bbox_init<<<1, 8, 0, ctx->stream>>>(bb);
    LO_CHECK_LAUNCH();
    bbox_kernel<<<grid_for(ctx, n, 256), 256, 0, ctx->stream>>>(xyz_dev, n, bb);
    LO_CHECK_LAUNCH();
    u64 h[7];
    fetch_small(ctx, bb, sizeof h);
    dfree(ctx, bb);
    std::memcpy(h, ctx->pinned_scratch, sizeof h);
    if (h[6] != ~0ull) {
        throw Error(LO_INVALID_ARGUMENT, "non-finite coordinate at point " + std::to_string(h[6]));
    }
    Disc d{};
    for (int a = 0; a < 6; ++a) d.cloud_box[a] = dbl_from_order_key(h[a]);
    // cubify (geometry.hpp:47-57): side = max extent, anchored at the min corner
    const double* b = d.cloud_box;
    const double side = std::max({b[3] - b[0], b[4] - b[1], b[5] - b[2]});
    for (int a = 0; a < 3; ++a) {
        d.box[a] = b[a];
        d.box[3 + a] = std::max(b[a] + side, b[3 + a]);
    }
    // Discretizer ctor (sfc.cpp:99-108) + axis_scale (sfc.cpp:77-80)
    for (int a = 0; a < 3; ++a) {
        const double extent = d.box[3 + a] - d.box[a];
        d.scale[a] = extent > 0.0 ? std::ldexp(1.0, level) / extent : 0.0;
    }
    return d;
}

// The three-level Hilbert table on this context's device (built from the CurveStepper closure,
// uploaded once per context).
static const u16* hilbert3_table(lo_context* ctx) {
    if (ctx->hilbert3) return static_cast<const u16*>(ctx->hilbert3);
    const CurveTables& t = curve_tables(LO_HILBERT);
    require(t.states == kH3States, LO_LOGIC_ERROR, "Hilbert table: unexpected state count");
    std::vector<u16> h(kH3Entries);
    for (int s0 = 0; s0 < kH3States; ++s0)
        for (u32 idx = 0; idx < 512; ++idx) {
            u32 st = static_cast<u32>(s0), code = 0;
            for (int l = 2; l >= 0; --l) {
                const u32 e = t.enc[st * 8 + ((idx >> (3 * l)) & 7u)];
                code = (code << 3) | (e & 7u);
                st = e >> 3;
            }
            h[s0 * 512 + idx] = static_cast<u16>(code | (st << 9));
        }
    void* d = nullptr;
    LO_CUDA(cudaMalloc(&d, h.size() * sizeof(u16)));
    LO_CUDA(cudaMemcpy(d, h.data(), h.size() * sizeof(u16), cudaMemcpyHostToDevice));
    ctx->hilbert3 = d;
    return static_cast<const u16*>(d);
}

static EncodeParams make_params(lo_context* ctx, const double box[6], const double scale[3], int level,
                                int curve) {
    EncodeParams p{};
    p.h3 = curve == LO_HILBERT ? hilbert3_table(ctx) : nullptr;
    for (int a = 0; a < 3; ++a) {
        p.lo[a] = box[a];
        p.hi[a] = box[3 + a];
        p.scale[a] = scale[a];
    }
    p.top = static_cast<double>((1ull << level) - 1);
    p.level = level;
    p.curve = curve;
    std::memcpy(p.enc, curve_tables(curve).enc, sizeof p.enc);
    return p;
}

// Sorts (codes, implicit original index) stably; writes sorted keys + perm.
// Digit bases per pass: exclusive scan of each pass's 256 counts (thread = pass).
__global__ void sort_bases(const u32* __restrict__ hist, u64* __restrict__ bases, int passes) {
    const int p = threadIdx.x;
    if (p >= passes) return;
    u64 s = 0;
    for (int b = 0; b < 256; ++b) {
        bases[p * 256 + b] = s;
        s += hist[p * 256 + b];
    }
}

void radix_sort(lo_context* ctx, u64* keys, u64 n, const u32* hist_host, int level,
                       u64* keys_sorted, u32* perm, const u32* hist_dev) {
    const int passes = (3 * level + 7) / 8;
    // digit bases per pass and the constant-digit skip (reorder.cpp:49)
    std::vector<int> run;
    std::vector<u64> bases(8 * 256, 0);
    for (int p = 0; p < passes; ++p) {
        bool trivial = false;
        u64 s = 0;
        for (int b = 0; b < 256; ++b) {
            const u32 c = hist_host[p * 256 + b];
            if (c == n) trivial = true;
            bases[p * 256 + b] = s;
            s += c;
        }
        if (!trivial) run.push_back(p);
    }
    if (run.empty()) {
        iota_u32<<<grid_for(ctx, n, 256), 256, 0, ctx->stream>>>(perm, n);
        LO_CHECK_LAUNCH();
        LO_CUDA(cudaMemcpyAsync(keys_sorted, keys, n * 8, cudaMemcpyDeviceToDevice, ctx->stream));
        return;
    }
    const int tiles = ceil_div(n, kSortTile);
    u64* dbase = dalloc_t<u64>(ctx, 8 * 256);
    if (hist_dev) {
        sort_bases<<<1, 32, 0, ctx->stream>>>(hist_dev, dbase, passes);
        LO_CHECK_LAUNCH();
    } else {
        LO_CUDA(cudaMemcpyAsync(dbase, bases.data(), bases.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
    }
    u64* status = dalloc_t<u64>(ctx, static_cast<size_t>(tiles) * 256);
    u32* counter = dalloc_t<u32>(ctx, 8);
    // one status memset per sort: each pass tags its words with its own epoch (i + 1); one memset for
    // the passes' tile counters too
    LO_CUDA(cudaMemsetAsync(status, 0, static_cast<size_t>(tiles) * 256 * 8, ctx->stream));
    LO_CUDA(cudaMemsetAsync(counter, 0, 8 * sizeof(u32), ctx->stream));
    u64* kalt = dalloc_t<u64>(ctx, n);
    u32* valt = dalloc_t<u32>(ctx, n);
    u32* vtmp = dalloc_t<u32>(ctx, n);
    // ping-pong so that the final pass lands in (keys_sorted, perm)
    const int np = static_cast<int>(run.size());
    const size_t smem = sizeof(SortSmem);
    if (!(ctx->smem_attrs & kAttrSort)) {
        LO_CUDA(cudaFuncSetAttribute(onesweep_pass<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
        ensure_smem_attr(ctx, kAttrSort, onesweep_pass<false>, smem);
    }
    const u64* kin = keys;
    const u32* vin = nullptr;
    for (int i = 0; i < np; ++i) {
        // pass i reads the previous pass's pair; the last pass lands in the outputs
        const bool last = i == np - 1;
        u64* kout = last ? keys_sorted : (i % 2 == 0 ? kalt : keys);
        u32* vout = last ? perm : (i % 2 == 0 ? valt : vtmp);
        if (i == 0)
            onesweep_pass<true><<<tiles, kSortThreads, smem, ctx->stream>>>(
                kin, nullptr, kout, vout, n, 8 * run[i], dbase + 256 * run[i], status, counter + i, i + 1);
        else
            onesweep_pass<false><<<tiles, kSortThreads, smem, ctx->stream>>>(
                kin, vin, kout, vout, n, 8 * run[i], dbase + 256 * run[i], status, counter + i, i + 1);
        LO_CHECK_LAUNCH();
        kin = kout;
        vin = vout;
    }
    dfree(ctx, dbase);
    dfree(ctx, status);
    dfree(ctx, counter);
    dfree(ctx, kalt);
    dfree(ctx, valt);
    dfree(ctx, vtmp);
}

// Curve order of arbitrary query points (clamped into the cloud's grid, so points outside the
// cube still get a position): codes + digit histograms, then the stable radix sort.
__global__ void __launch_bounds__(256) query_codes(const double* __restrict__ x, const double* __restrict__ y,
                                                   const double* __restrict__ z, u64 n, EncodeParams p,
                                                   u64* __restrict__ codes, u32* __restrict__ hist) {
    __shared__ u8 enc[32 * 8];
    __shared__ __align__(16) u16 h3[kH3Entries];
    __shared__ u32 h[8 * 256];
    for (int i = threadIdx.x; i < 32 * 8; i += blockDim.x) enc[i] = p.enc[i];
    load_h3(h3, p);
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) h[i] = 0;
    __syncthreads();
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u32 cx = axis_cell(x[i], p.lo[0], p.scale[0], p.top);
        const u32 cy = axis_cell(y[i], p.lo[1], p.scale[1], p.top);
        const u32 cz = axis_cell(z[i], p.lo[2], p.scale[2], p.top);
        const u64 code = encode_cell(cx, cy, cz, p.level, p.curve, enc, h3);
        codes[i] = code;
#pragma unroll
        for (int b = 0; b < 8; ++b) atomicAdd(&h[b * 256 + ((code >> (8 * b)) & 0xff)], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x)
        if (h[i]) atomicAdd(&hist[i], h[i]);
}

u32* sort_points_sfc(lo_context* ctx, const lo_coded* c, const double* x, const double* y, const double* z,
                     u64 m) {
    if (m == 0) return nullptr;
    u64* codes = dalloc_t<u64>(ctx, m);
    u64* sorted = nullptr;
    u32* hist = nullptr;
    u32* pos = nullptr;
    try {
        sorted = dalloc_t<u64>(ctx, m);
        hist = dalloc_t<u32>(ctx, 8 * 256);
        pos = dalloc_t<u32>(ctx, m);
        LO_CUDA(cudaMemsetAsync(hist, 0, 8 * 256 * 4, ctx->stream));
        const EncodeParams p = make_params(ctx, c->disc_box, c->scale, c->level, c->curve);
        query_codes<<<std::min(grid_for(ctx, m, 256), ctx->sm_count * 4), 256, 0, ctx->stream>>>(x, y, z, m, p,
                                                                                              codes, hist);
        LO_CHECK_LAUNCH();
        std::vector<u32> hh(8 * 256);
        fetch_small(ctx, hist, 8 * 256 * 4);
        std::memcpy(hh.data(), ctx->pinned_scratch, 8 * 256 * 4);
        radix_sort(ctx, codes, m, hh.data(), c->level, sorted, pos, hist);
    } catch (...) {
        dfree(ctx, codes), dfree(ctx, sorted), dfree(ctx, hist), dfree(ctx, pos);
        throw;
    }
    dfree(ctx, codes), dfree(ctx, sorted), dfree(ctx, hist);
    return pos;
}

lo_coded* reorder_device(lo_context* ctx, const double* xyz, u64 n, int curve, int level) {
    require(n > 0, LO_INVALID_ARGUMENT, "reorder_cloud: empty cloud");
    require(n <= 0xffffffffull, LO_INVALID_ARGUMENT,
            "reorder_cloud: cloud exceeds 32-bit index space");
    require(level >= 0 && level <= kMaxLevel, LO_INVALID_ARGUMENT, "level out of range");
    require(curve == LO_MORTON || curve == LO_HILBERT, LO_INVALID_ARGUMENT, "unknown curve");
    stage_begin(ctx, "bbox");
    const Disc disc = compute_disc(ctx, xyz, n, level);
    stage_end(ctx);

    auto* c = new lo_coded;
    c->ctx = ctx;
    c->n = n;
    c->curve = curve;
    c->level = level;
    std::memcpy(c->cloud_box, disc.cloud_box, sizeof disc.cloud_box);
    std::memcpy(c->disc_box, disc.box, sizeof disc.box);
    std::memcpy(c->scale, disc.scale, sizeof disc.scale);
    try {
        stage_begin(ctx, "encode");
        u64* codes = dalloc_t<u64>(ctx, n);
        u32* hist = dalloc_t<u32>(ctx, 8 * 256 + 1);
        LO_CUDA(cudaMemsetAsync(hist, 0, (8 * 256 + 1) * 4, ctx->stream));
        const EncodeParams p = make_params(ctx, disc.box, disc.scale, level, curve);
        encode_kernel<true><<<grid_for(ctx, n, 256, encode_per_sm()), 256, 0, ctx->stream>>>(
            xyz, n, p, codes, hist, hist + 8 * 256);
        LO_CHECK_LAUNCH();
        stage_end(ctx);
        std::vector<u32> hh(8 * 256 + 1);
        fetch_small(ctx, hist, hh.size() * 4);
        std::memcpy(hh.data(), ctx->pinned_scratch, hh.size() * 4);
        require(hh[8 * 256] == 0, LO_DOMAIN_ERROR, "point outside discretizer bounds");

        stage_begin(ctx, "sort");
        c->codes = dalloc_t<u64>(ctx, n);
        c->perm = dalloc_t<u32>(ctx, n);
        radix_sort(ctx, codes, n, hh.data(), level, c->codes, c->perm, hist);
        stage_end(ctx);
        dfree(ctx, codes);
        dfree(ctx, hist);

        stage_begin(ctx, "gather");
        c->x = dalloc_t<double>(ctx, n);
        c->y = dalloc_t<double>(ctx, n);
        c->z = dalloc_t<double>(ctx, n);
        c->pf = dalloc_t<float4>(ctx, n);
        set_origin(c);
        gather_soa<<<grid_for(ctx, n, 256), 256, 0, ctx->stream>>>(
            xyz, c->perm, n, c->x, c->y, c->z, c->pf, c->origin[0], c->origin[1], c->origin[2]);
        LO_CHECK_LAUNCH();
        stage_end(ctx);
        sync(ctx);
    } catch (...) {
        dfree(ctx, c->codes);
        dfree(ctx, c->perm);
        dfree(ctx, c->x);
        dfree(ctx, c->y);
        dfree(ctx, c->z);
        dfree(ctx, c->pf);
        delete c;
        throw;
    }
    return c;
}

}  // namespace lo

using namespace lo;

extern "C" {

int lo_compute_codes(lo_context* ctx, const double* xyz_host, uint64_t n, int curve, int level,
                     const double* disc_box, uint64_t* codes_host) {
    return api_ctx(ctx, [&] {
        require(n > 0, LO_INVALID_ARGUMENT, "compute_codes: empty cloud");
        require(level >= 0 && level <= kMaxLevel, LO_INVALID_ARGUMENT, "level out of range");
        double* xyz = dalloc_t<double>(ctx, 3 * n);
        u64* codes = dalloc_t<u64>(ctx, n);
        u32* err = dalloc_t<u32>(ctx, 1);
        LO_CUDA(cudaMemsetAsync(err, 0, 4, ctx->stream));
        LO_CUDA(cudaMemcpyAsync(xyz, xyz_host, 24 * n, cudaMemcpyHostToDevice, ctx->stream));
        double box[6], scale[3];
        if (disc_box) {
            for (int a = 0; a < 3; ++a) {
                require(disc_box[a] <= disc_box[3 + a], LO_INVALID_ARGUMENT, "inverted bounding box");
                const double extent = disc_box[3 + a] - disc_box[a];
                scale[a] = extent > 0.0 ? std::ldexp(1.0, level) / extent : 0.0;
            }
            std::memcpy(box, disc_box, sizeof box);
        } else {
            const Disc d = compute_disc(ctx, xyz, n, level);
            std::memcpy(box, d.box, sizeof box);
            std::memcpy(scale, d.scale, sizeof scale);
        }
        const EncodeParams p = make_params(ctx, box, scale, level, curve);
        encode_kernel<false><<<grid_for(ctx, n, 256, encode_per_sm()), 256, 0, ctx->stream>>>(xyz, n, p, codes,
                                                                                nullptr, err);
        LO_CHECK_LAUNCH();
        LO_CUDA(cudaMemcpyAsync(codes_host, codes, 8 * n, cudaMemcpyDeviceToHost, ctx->stream));
        const u32 e = read_scalar(ctx, err);
        dfree(ctx, xyz);
        dfree(ctx, codes);
        dfree(ctx, err);
        sync(ctx);
        require(e == 0, LO_DOMAIN_ERROR, "point outside discretizer bounds");
    });
}

int lo_encode_cells(lo_context* ctx, const uint32_t* cells_host, uint64_t n, int curve, int level,
                    uint64_t* codes_host) {
    return api_ctx(ctx, [&] {
        require(level >= 0 && level <= kMaxLevel, LO_INVALID_ARGUMENT, "level out of range");
        if (n == 0) return;
        u32* cells = dalloc_t<u32>(ctx, 3 * n);
        u64* codes = dalloc_t<u64>(ctx, n);
        LO_CUDA(cudaMemcpyAsync(cells, cells_host, 12 * n, cudaMemcpyHostToDevice, ctx->stream));
        const double box[6] = {0, 0, 0, 1, 1, 1}, scale[3] = {0, 0, 0};
        const EncodeParams p = make_params(ctx, box, scale, level, curve);
        encode_cells_kernel<<<grid_for(ctx, n, 256), 256, 0, ctx->stream>>>(cells, n, level, curve,
                                                                            p, codes);
        LO_CHECK_LAUNCH();
        LO_CUDA(cudaMemcpyAsync(codes_host, codes, 8 * n, cudaMemcpyDeviceToHost, ctx->stream));
        dfree(ctx, cells);
        dfree(ctx, codes);
        sync(ctx);
    });
}

int lo_decode_codes(lo_context* ctx, const uint64_t* codes_host, uint64_t n, int curve, int level,
                    uint32_t* cells_host) {
    return api_ctx(ctx, [&] {
        require(level >= 0 && level <= kMaxLevel, LO_INVALID_ARGUMENT, "level out of range");
        if (n == 0) return;
        u64* codes = dalloc_t<u64>(ctx, n);
        u32* cells = dalloc_t<u32>(ctx, 3 * n);
        LO_CUDA(cudaMemcpyAsync(codes, codes_host, 8 * n, cudaMemcpyHostToDevice, ctx->stream));
        decode_codes_kernel<<<grid_for(ctx, n, 256), 256, 0, ctx->stream>>>(
            codes, n, level, curve_tables(curve), cells);
        LO_CHECK_LAUNCH();
        LO_CUDA(cudaMemcpyAsync(cells_host, cells, 12 * n, cudaMemcpyDeviceToHost, ctx->stream));
        dfree(ctx, codes);
        dfree(ctx, cells);
        sync(ctx);
    });
}

int lo_reorder_device(lo_context* ctx, const double* xyz_dev, uint64_t n, int curve, int level,
                      lo_coded** out) {
    return api_ctx(ctx, [&] { *out = reorder_device(ctx, xyz_dev, n, curve, level); });
}

int lo_reorder(lo_context* ctx, const double* xyz_host, uint64_t n, int curve, int level,
               lo_coded** out) {
    return api_ctx(ctx, [&] {
        require(n > 0, LO_INVALID_ARGUMENT, "reorder_cloud: empty cloud");
        double* xyz = dalloc_t<double>(ctx, 3 * n);
        try {
            stage_begin(ctx, "h2d");
            LO_CUDA(cudaMemcpyAsync(xyz, xyz_host, 24 * n, cudaMemcpyHostToDevice, ctx->stream));
            stage_end(ctx);
            *out = reorder_device(ctx, xyz, n, curve, level);
        } catch (...) {
            dfree(ctx, xyz);
            throw;
        }
        dfree(ctx, xyz);
    });
}

int lo_coded_info_get(const lo_coded* c, lo_coded_info* out) {
    return api([&] {
        require(c != nullptr, LO_INVALID_ARGUMENT, "null coded cloud");
        out->n = c->n;
        out->curve = c->curve;
        out->level = c->level;
        std::memcpy(out->disc_box, c->disc_box, sizeof c->disc_box);
        std::memcpy(out->cloud_box, c->cloud_box, sizeof c->cloud_box);
        std::memcpy(out->scale, c->scale, sizeof c->scale);
    });
}

int lo_coded_download(lo_context* ctx, const lo_coded* c, double* xyz_host, uint64_t* codes_host,
                      uint32_t* perm_host) {
    return api_ctx(ctx, [&] {
        const u64 n = c->n;
        if (xyz_host) {
            double* aos = dalloc_t<double>(ctx, 3 * n);
            interleave_aos<<<grid_for(ctx, n, 256), 256, 0, ctx->stream>>>(c->x, c->y, c->z, n, aos);
            LO_CHECK_LAUNCH();
            LO_CUDA(cudaMemcpyAsync(xyz_host, aos, 24 * n, cudaMemcpyDeviceToHost, ctx->stream));
            dfree(ctx, aos);
        }
        if (codes_host)
            LO_CUDA(cudaMemcpyAsync(codes_host, c->codes, 8 * n, cudaMemcpyDeviceToHost, ctx->stream));
        if (perm_host)
            LO_CUDA(cudaMemcpyAsync(perm_host, c->perm, 4 * n, cudaMemcpyDeviceToHost, ctx->stream));
        sync(ctx);
    });
}

int lo_coded_device_ptrs(const lo_coded* c, const double** x, const double** y, const double** z,
                         const uint64_t** codes, const uint32_t** perm) {
    return api([&] {
        if (x) *x = c->x;
        if (y) *y = c->y;
        if (z) *z = c->z;
        if (codes) *codes = c->codes;
        if (perm) *perm = c->perm;
    });
}

int lo_coded_destroy(lo_coded* c) {
    if (!c) return LO_OK;
    return api_ctx(c->ctx, [&] {
        lo_context* ctx = c->ctx;
        if (c->reader) {  // a broadcast / peer copy may still read the buffers: free behind it
            LO_CUDA(cudaStreamWaitEvent(ctx->stream, c->reader, 0));
            cudaEventDestroy(c->reader);
        }
        dfree(ctx, c->x);
        dfree(ctx, c->y);
        dfree(ctx, c->z);
        dfree(ctx, c->codes);
        dfree(ctx, c->perm);
        dfree(ctx, c->pf);
        delete c;
    });
}

int lo_coded_create_empty(lo_context* ctx, const lo_coded_info* info, lo_coded** out) {
    return api_ctx(ctx, [&] {
        require(info && info->n > 0 && info->n <= 0xffffffffull, LO_INVALID_ARGUMENT,
                "coded cloud header: bad size");
        auto* c = new lo_coded;
        c->ctx = ctx;
        c->n = info->n;
        c->curve = info->curve;
        c->level = info->level;
        std::memcpy(c->disc_box, info->disc_box, sizeof c->disc_box);
        std::memcpy(c->cloud_box, info->cloud_box, sizeof c->cloud_box);
        std::memcpy(c->scale, info->scale, sizeof c->scale);
        set_origin(c);  // pf is rebuilt lazily from the broadcast coordinates
        try {
            c->x = dalloc_t<double>(ctx, c->n);
            c->y = dalloc_t<double>(ctx, c->n);
            c->z = dalloc_t<double>(ctx, c->n);
            c->codes = dalloc_t<u64>(ctx, c->n);
            c->perm = dalloc_t<u32>(ctx, c->n);
            sync(ctx);
        } catch (...) {
            dfree(ctx, c->x), dfree(ctx, c->y), dfree(ctx, c->z), dfree(ctx, c->codes), dfree(ctx, c->perm);
            delete c;
            throw;
        }
        *out = c;
    });
}

int lo_invert_permutation(lo_context* ctx, const uint32_t* perm_host, uint64_t n, uint32_t* inv_host) {
    return api_ctx(ctx, [&] {
        if (n == 0) return;
        u32* p = dalloc_t<u32>(ctx, n);
        u32* q = dalloc_t<u32>(ctx, n);
        LO_CUDA(cudaMemcpyAsync(p, perm_host, 4 * n, cudaMemcpyHostToDevice, ctx->stream));
        invert_perm_kernel<<<grid_for(ctx, n, 256), 256, 0, ctx->stream>>>(p, n, q);
        LO_CHECK_LAUNCH();
        LO_CUDA(cudaMemcpyAsync(inv_host, q, 4 * n, cudaMemcpyDeviceToHost, ctx->stream));
        dfree(ctx, p);
        dfree(ctx, q);
        sync(ctx);
    });
}

}  // extern "C"
