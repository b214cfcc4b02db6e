// radius_pt.cuh -- radius walk with lane = candidate point (K6 count / fill), used by radius.cu.
//
// Same traversal as radius_float.cuh (warp = 32 consecutive queries, child-parallel expansion
// with per-group pruning), but leaves are not tested lane = query.  The points of every visited
// leaf are appended, in code order, to a dense 32-slot shared-memory buffer; the buffer also
// records which of the 32 queries reach any of its leaves.  A full buffer is processed with
// lane j = buffer point j: for each interested query (two at a time, packed FP32 f32x2 math)
// the warp ballots membership, so
//   * no lane idles on small terrain leaves (~10 points) -- every slot is a real candidate,
//   * the fill pass writes query L's members of the buffer with ONE coalesced store
//     (position = row cursor + popc(mask below the lane)), no per-member loops,
//   * rows stay ascending: buffers follow the DFS code order and slots keep point order.
// Uncertainty-band points (search_common.cuh) are decided by the exact FP64 predicate.
#pragma once

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "radius_float.cuh"

namespace lo {

#ifndef LO_PT_WARPS
#define LO_PT_WARPS 4
#endif
// count-kernel blocks per SM (__launch_bounds__ minimum; the persistent grid is sm_count x this).
// 10 (48 registers, a 44-byte spill) beats 6 / 7 / 8 / 9 / 12 on cfg1, cfg3 and cfg4: the walk is
// latency bound and the extra resident warps hide more of it than the spill costs
// (cfg3 count 30.8 / 30.3 / 28.9 / 28.1 / 27.2 / 29.1 ms, profiles/r3/count_minb_ab.log).
#ifndef LO_PT_MINB
#define LO_PT_MINB 10
#endif
constexpr int kPtWarps = LO_PT_WARPS;
#ifndef LO_PT_PREFILTER
#define LO_PT_PREFILTER 1
#endif
// LO_PT_STREAM=1: the walk queues up to 32 kept leaves and streams their points 32 at a time across
// leaf boundaries, the next 32 prefetched by cp.async while the current ones are filtered.  Measured
// slower (cfg3 count 33.8 -> 35.5 ms, cfg1 r = 3 4.98 -> 5.23 ms): the stream lookup costs more than
// the per-leaf load latency it hides.
#ifndef LO_PT_STREAM
#define LO_PT_STREAM 0
#endif
#ifndef LO_PT_UNROLL_FULL
#define LO_PT_UNROLL_FULL 1
#endif
constexpr int kPtThreads = 32 * kPtWarps;

struct PtShared {
    u32 stack[kStackCap];
#if LO_PT_STREAM
    u32 lbeg[32];        // queued leaves (walk order): first point, point count, wanting queries
    u32 lsize[32];
    u32 lwant[32];
    float4 pre[2][32];   // streamed candidate points (FP32, cloud frame), double-buffered
#endif
    float tbox[6];       // the tile's FP32 query box (lo xyz, hi xyz)
    u32 bix[32];         // candidate point indices, staged per leaf (loaded per buffer)
    float4 qf[32];       // queries, FP32 relative to the cloud origin (walk: node-box tests)
    // queries, FP32 relative to the tile origin (point tests), SoA: (q[2p], q[2p+1]) loads as
    // one f32x2
    __align__(16) float qx[32];
    __align__(16) float qy[32];
    __align__(16) float qz[32];
    double qd[32][3];    // queries, FP64 (band decisions)
    __align__(16) u32 msk[32];  // count pass: membership ballot of query L for the current buffer
};

// Decide band lanes exactly; returns the corrected membership ballot for query L.
template <int SHAPE>
__device__ __forceinline__ u32 band_fix(u32 in, u32 band, const PtShared& S, int L, int lane,
                                        u32 idx, const double* __restrict__ px,
                                        const double* __restrict__ py, const double* __restrict__ pz,
                                        double r, double r2) {
    bool m = false;
    if ((band >> lane) & 1u)
        m = contains<SHAPE>(S.qd[L][0], S.qd[L][1], S.qd[L][2], r, r2, px[idx], py[idx], pz[idx]);
    return in | __ballot_sync(~0u, m);
}

// Tests the buffer's `fill` points (lane j = slot j) against the interested queries, taken as
// fixed pairs (2p, 2p+1) so both query coordinates arrive as one packed f32x2 load.  Lane L
// keeps query L's count (count pass) or its CSR cursor relative to the tile's first row
// (fill pass) in a register.
template <int SHAPE, bool FILL>
__device__ __forceinline__ void process_buffer(PtShared& S, const float4 P, u32 fill, u32 qmask, int lane,
                                               float lo_thr, float hi_thr,
                                               const double* __restrict__ px,
                                               const double* __restrict__ py,
                                               const double* __restrict__ pz, double r,
                                               double r2, u32* __restrict__ out_tile, u32& mine,
                                               u32& mymask) {
    constexpr bool kPacked = SHAPE == LO_SPHERE || SHAPE == LO_CIRCLE;
    // slots >= fill hold +INF (staged that way), so they are never members; a query that is
    // disjoint from every leaf of the buffer has d2_f >= near2_f >= t_hi for all its points,
    // so testing it anyway yields an empty ballot -- no per-query interest masks are needed.
    const u32 idx = __float_as_uint(P.w);
    const u64 PX = pack2(P.x, P.x), PY = pack2(P.y, P.y), PZ = pack2(P.z, P.z);
    const u32 lt = (1u << lane) - 1u;
    const u32 lo_bits = __float_as_uint(lo_thr);
    const u32 band_bits = __float_as_uint(hi_thr) - lo_bits;
    if (!FILL && kPacked) {
        // count pass: four queries (two packed pairs) per iteration -- one 16-byte mask store and one
        // loop step for four membership ballots.  The FP32 band is only tracked per lane in the loop
        // (min over its values of bits(v) - bits(lo)); one vote after the loop decides whether any
        // pair fell in the band, and only then are the quads redone with the exact FP64 decisions.
        const u32 qm0 = (qmask | (qmask >> 1) | (qmask >> 2) | (qmask >> 3)) & 0x11111111u;
        S.msk[lane] = 0u;
        __syncwarp();
        auto quad = [&](int b, float* v) {
            const float4 X = *reinterpret_cast<const float4*>(&S.qx[b]);
            const float4 Y = *reinterpret_cast<const float4*>(&S.qy[b]);
            const u64 dxa = fsub2(PX, pack2(X.x, X.y)), dxb = fsub2(PX, pack2(X.z, X.w));
            const u64 dya = fsub2(PY, pack2(Y.x, Y.y)), dyb = fsub2(PY, pack2(Y.z, Y.w));
            u64 da = fmul2(dxa, dxa), db = fmul2(dxb, dxb);
            da = ffma2(dya, dya, da);
            db = ffma2(dyb, dyb, db);
            if (SHAPE == LO_SPHERE) {
                const float4 Z = *reinterpret_cast<const float4*>(&S.qz[b]);
                const u64 dza = fsub2(PZ, pack2(Z.x, Z.y)), dzb = fsub2(PZ, pack2(Z.z, Z.w));
                da = ffma2(dza, dza, da);
                db = ffma2(dzb, dzb, db);
            }
            unpack2(da, v[0], v[1]);
            unpack2(db, v[2], v[3]);
        };
        u32 band_min = 0xffffffffu;
        auto quad_pass = [&](int b) {
            float v[4];
            quad(b, v);
            u32 in[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) in[t] = __ballot_sync(~0u, v[t] < lo_thr);
            const u32 w01 = min(__float_as_uint(v[0]) - lo_bits, __float_as_uint(v[1]) - lo_bits);
            const u32 w23 = min(__float_as_uint(v[2]) - lo_bits, __float_as_uint(v[3]) - lo_bits);
            band_min = min(band_min, min(w01, w23));
            if (lane == 0) *reinterpret_cast<uint4*>(&S.msk[b]) = make_uint4(in[0], in[1], in[2], in[3]);
        };
#if LO_PT_UNROLL_FULL
        if (qm0 == 0x11111111u) {  // every query interested (the common case): straight-line, static offsets
#pragma unroll
            for (int q = 0; q < 8; ++q) quad_pass(4 * q);
        } else
#endif
        {
            for (u32 qm = qm0; qm; qm &= qm - 1) quad_pass(__ffs(qm) - 1);  // b = 4q
        }
        if (__any_sync(~0u, band_min < band_bits)) {  // rare: band points, exact FP64 decides
            for (u32 qm = qm0; qm; qm &= qm - 1) {
                const int b = __ffs(qm) - 1;
                float v[4];
                quad(b, v);
                u32 in[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    in[t] = __ballot_sync(~0u, v[t] < lo_thr);
                    const u32 h = __ballot_sync(~0u, v[t] < hi_thr);
                    if (h ^ in[t]) in[t] = band_fix<SHAPE>(in[t], h ^ in[t], S, b + t, lane, idx, px, py, pz, r, r2);
                }
                if (lane == 0) *reinterpret_cast<uint4*>(&S.msk[b]) = make_uint4(in[0], in[1], in[2], in[3]);
            }
        }
        __syncwarp();
        mymask = S.msk[lane];
        return;
    }
    u32 pm = (qmask | (qmask >> 1)) & 0x55555555u;  // bit 2p: pair p has an interested query
    if (!FILL) {
        S.msk[lane] = 0u;
        __syncwarp();
    }
    while (pm) {
        const int b = __ffs(pm) - 1;  // = 2p
        pm &= pm - 1;
        float v0, v1;
        if (kPacked) {
            const u64 dx = fsub2(PX, *reinterpret_cast<const u64*>(&S.qx[b]));
            const u64 dy = fsub2(PY, *reinterpret_cast<const u64*>(&S.qy[b]));
            u64 d2 = fmul2(dx, dx);
            d2 = ffma2(dy, dy, d2);
            if (SHAPE == LO_SPHERE) {
                const u64 dz = fsub2(PZ, *reinterpret_cast<const u64*>(&S.qz[b]));
                d2 = ffma2(dz, dz, d2);
            }
            unpack2(d2, v0, v1);
        } else {
            v0 = metric_f<SHAPE>(make_float4(S.qx[b], S.qy[b], S.qz[b], 0.f), P);
            v1 = metric_f<SHAPE>(make_float4(S.qx[b + 1], S.qy[b + 1], S.qz[b + 1], 0.f), P);
        }
        u32 in0 = __ballot_sync(~0u, v0 < lo_thr);
        u32 in1 = __ballot_sync(~0u, v1 < lo_thr);
        // band lo <= v < hi as one unsigned range test on the bits (v >= 0 or NaN, lo > 0)
        if (__any_sync(~0u, (__float_as_uint(v0) - lo_bits < band_bits) |
                                (__float_as_uint(v1) - lo_bits < band_bits))) {
            // rare: band points, exact FP64 decides
            const u32 h0 = __ballot_sync(~0u, v0 < hi_thr);
            const u32 h1 = __ballot_sync(~0u, v1 < hi_thr);
            if (h0 ^ in0) in0 = band_fix<SHAPE>(in0, h0 ^ in0, S, b, lane, idx, px, py, pz, r, r2);
            if (h1 ^ in1) in1 = band_fix<SHAPE>(in1, h1 ^ in1, S, b + 1, lane, idx, px, py, pz, r, r2);
        }
        if (FILL) {
            const u32 c0 = __shfl_sync(~0u, mine, b);
            const u32 c1 = __shfl_sync(~0u, mine, b + 1);
            if ((in0 >> lane) & 1u) out_tile[c0 + __popc(in0 & lt)] = idx;
            if ((in1 >> lane) & 1u) out_tile[c1 + __popc(in1 & lt)] = idx;
            mine += lane == b ? __popc(in0) : (lane == b + 1 ? __popc(in1) : 0u);
        } else if (lane == 0) {
            // query L's membership mask of this buffer (count + record)
            *reinterpret_cast<uint2*>(&S.msk[b]) = make_uint2(in0, in1);
        }
    }
    if (!FILL) {
        __syncwarp();
        mymask = S.msk[lane];
    }
}

constexpr u32 kRecOverflow = 0xffffffffu;
constexpr u32 kRecChunk = 1024;  // records per warp chunk (256 KB)

// Count-pass records, packed: each warp takes chunks of kRecChunk records from a bump
// allocator and appends its tiles' records contiguously; tile t's records start at record
// rec_off[t] and number rec_n[t] (kRecOverflow: not recorded -> fill-walk fallback).
struct RecPool {
    u32* pool = nullptr;    // 64 words per record: 32 slot indices, 32 query masks
    u64 pool_recs = 0;
    u64* alloc = nullptr;   // bump counter (records)
    u32 cap = 0;            // max records per tile
    u32* rec_n = nullptr;   // [tiles]
    u64* rec_off = nullptr; // [tiles]
};

// Fill pass by replay of the count pass's records: record b of a tile holds the 32 slot indices
// of one processed buffer and, per query lane, its membership mask.  The tile's records are
// staged in shared memory and the rows are written one after the other: row L takes its members
// of buffer b with one coalesced store at consecutive CSR slots, so every output line is
// completed while it is hot in L2 (writing buffer-major across all 32 rows left ~10^4 tiles'
// lines half-written and cost read-modify-write traffic).  No walk, no re-tested points.
constexpr int kReplayWarps = 4;

// Buffer-major replay for short rows (small radii): per record, one coalesced store per query
// with members; the few, short rows of a tile stay within a handful of lines.
static __global__ void __launch_bounds__(128) radius_replay_bm_kernel(
    RecPool rp, u64 m, const u64* __restrict__ offsets, u32* __restrict__ out,
    u32* __restrict__ overflow_list, u32* __restrict__ overflow_n) {
    const int lane = threadIdx.x & 31;
    const u32 lt = (1u << lane) - 1u;
    const u64 ntiles = (m + 31) / 32;
    for (u64 tile = (static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; tile < ntiles;
         tile += (static_cast<u64>(gridDim.x) * blockDim.x) >> 5) {
        const u32 n = rp.rec_n[tile];
        if (n == kRecOverflow) {
            if (lane == 0) overflow_list[atomicAdd(overflow_n, 1u)] = static_cast<u32>(tile);
            continue;
        }
        const u64 qi = tile * 32 + lane;
        const u64 tbase = offsets[tile * 32];
        u32* out_tile = out + tbase;
        u32 cursor = qi < m ? static_cast<u32>(offsets[qi] - tbase) : 0u;
        asm("" : "+l"(out_tile));  // keep the stores as 32-bit offsets from one base
        const u32* R = rp.pool + rp.rec_off[tile] * 64;
        // record b + 1 is loaded while record b is written (the loads were exposed before)
        u32 idx = 0, mk = 0;
        if (n) idx = __ldg(R + lane), mk = __ldg(R + 32 + lane);
        for (u32 b = 0; b < n; ++b) {
            u32 idx_n = 0, mk_n = 0;
            if (b + 1 < n) idx_n = __ldg(R + 64 * (b + 1) + lane), mk_n = __ldg(R + 64 * (b + 1) + 32 + lane);
            unsigned nz = __ballot_sync(~0u, mk != 0);
            while (nz) {
                const int L = __ffs(nz) - 1;
                nz &= nz - 1;
                const u32 mL = __shfl_sync(~0u, mk, L);
                const u32 cL = __shfl_sync(~0u, cursor, L);
                if ((mL >> lane) & 1u) __stcg(out_tile + (cL + __popc(mL & lt)), idx);
            }
            cursor += __popc(mk);
            idx = idx_n, mk = mk_n;
        }
    }
}

// Row-major replay for long rows.  The tile's records (read exactly once, streamed) are staged in
// this warp's shared memory 32 at a time: slot indices as [b][32], masks as [b][33] so that lane b
// reading row L's mask of buffer b is bank-conflict free.  Per row, lane b holds the row's mask of
// buffer b; a warp scan of the popcounts gives every buffer's CSR start, and the write loop is two
// shuffles, one shared load and one coalesced store per (row, buffer with members).
constexpr u32 kReplayMaskStride = 33;
#ifndef LO_REPLAY_ROWS
#define LO_REPLAY_ROWS 4
#endif
#ifndef LO_REPLAY_BLOCKS
#define LO_REPLAY_BLOCKS 5
#endif
constexpr int kReplayRows = LO_REPLAY_ROWS;  // rows per write pass (even)
constexpr int kReplayBlocks = LO_REPLAY_BLOCKS;
constexpr size_t kReplayWarpWords = 32 * 32 + 32 * kReplayMaskStride + 32 * 2 * kReplayRows;
constexpr size_t kReplaySmem = kReplayWarps * kReplayWarpWords * 4;

static __global__ void __launch_bounds__(32 * kReplayWarps, kReplayBlocks) radius_replay_kernel(
    RecPool rp, u64 m, const u64* __restrict__ offsets, u32* __restrict__ out,
    u32* __restrict__ overflow_list, u32* __restrict__ overflow_n) {
    extern __shared__ __align__(16) u32 replay_smem[];
    const u32* __restrict__ rec_n = rp.rec_n;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const u32 lt = (1u << lane) - 1u;
    u32* I = replay_smem + w * kReplayWarpWords;  // [32][32] slot indices
    u32* M = I + 32 * 32;                         // [32][33] per-row masks
    // per buffer (mask, CSR start) of the two rows in flight: the write loop reads them with one
    // broadcast 8-byte shared load instead of two shuffles (the MIO pipe is the step's limit)
    uint4* RM = reinterpret_cast<uint4*>(M + 32 * kReplayMaskStride);  // [b][r/2] = (m, p) of rows r, r+1
    const u32 rmh = static_cast<u32>(__cvta_generic_to_shared(RM));
    const u32 ih = static_cast<u32>(__cvta_generic_to_shared(I + lane));
    const u64 ntiles = (m + 31) / 32;
    for (u64 tile = static_cast<u64>(blockIdx.x) * kReplayWarps + w; tile < ntiles;
         tile += static_cast<u64>(gridDim.x) * kReplayWarps) {
        const u32 n = rec_n[tile];
        if (n == kRecOverflow) {
            if (lane == 0) overflow_list[atomicAdd(overflow_n, 1u)] = static_cast<u32>(tile);
            continue;
        }
        const u64 qi = tile * 32 + lane;
        const u64 tbase = offsets[tile * 32];
        u32 cursor = qi < m ? static_cast<u32>(offsets[qi] - tbase) : 0u;  // lane L: row L
        const u32 total = qi < m ? static_cast<u32>(offsets[qi + 1] - offsets[qi]) : 0u;
        const unsigned rows_all = __ballot_sync(~0u, total != 0);
        u32* out_tile = out + tbase;
        asm("" : "+l"(out_tile));  // keep the row stores as 32-bit offsets from one base
        const uint4* R4 = reinterpret_cast<const uint4*>(rp.pool + rp.rec_off[tile] * 64);
        for (u32 h0 = 0; h0 < n; h0 += 32) {
            const u32 nh = min(32u, n - h0);
            const u32 nv = nh * 16;
            const uint4* Rh = R4 + h0 * 16;
            __syncwarp();
            for (u32 i0 = 0; i0 < nv; i0 += 128) {
                uint4 v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const u32 i = i0 + u * 32 + lane;
                    if (i < nv) v[u] = __ldcs(Rh + i);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const u32 i = i0 + u * 32 + lane;
                    if (i < nv) {
                        const u32 b = i >> 4, part = i & 15;
                        if (part < 8) {
                            *reinterpret_cast<uint4*>(I + b * 32 + part * 4) = v[u];
                        } else {
                            u32* d = M + b * kReplayMaskStride + (part - 8) * 4;
                            d[0] = v[u].x, d[1] = v[u].y, d[2] = v[u].z, d[3] = v[u].w;
                        }
                    }
                }
            }
            __syncwarp();
            // kReplayRows rows per pass: their scans are independent chains, and the write loop runs
            // once over the union of their buffers -- neighbouring queries draw on mostly the same
            // buffers, so one index load serves up to kReplayRows stores
            unsigned rows = rows_all;
            u32 adv = 0;  // lane L: row L's members in this half
            const bool in = static_cast<u32>(lane) < nh;
            while (rows) {
                int Ls[kReplayRows];
                u32 mk[kReplayRows], sc[kReplayRows], pk[kReplayRows];
                bool val[kReplayRows];
                u32 any = 0;
#pragma unroll
                for (int r = 0; r < kReplayRows; ++r) {
                    val[r] = rows != 0;
                    Ls[r] = val[r] ? __ffs(rows) - 1 : 0;
                    rows &= rows - 1;
                    mk[r] = in && val[r] ? M[lane * kReplayMaskStride + Ls[r]] : 0u;
                    sc[r] = __popc(mk[r]);
                    any |= mk[r];
                }
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
                    for (int r = 0; r < kReplayRows; ++r) {
                        const u32 t = __shfl_up_sync(~0u, sc[r], o);
                        if (lane >= o) sc[r] += t;
                    }
                }
#pragma unroll
                for (int r = 0; r < kReplayRows; ++r) {
                    pk[r] = __shfl_sync(~0u, cursor, Ls[r]) + sc[r] - __popc(mk[r]);  // exclusive starts
                    const u32 tot = __shfl_sync(~0u, sc[r], 31);
                    if (val[r] && lane == Ls[r]) adv = tot;
                }
                unsigned nz = __ballot_sync(~0u, any != 0);
                __syncwarp();  // the previous pass's write loop is done with RM
#pragma unroll
                for (int r = 0; r < kReplayRows; r += 2) RM[lane * (kReplayRows / 2) + r / 2] = make_uint4(mk[r], pk[r], mk[r + 1], pk[r + 1]);
                __syncwarp();
                auto step = [&](int b) {
                    u32 idx;
                    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(idx) : "r"(ih + b * 128) : "memory");
#pragma unroll
                    for (int r = 0; r < kReplayRows; r += 2) {
                        u32 mA, pA, mB, pB;
                        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                                     : "=r"(mA), "=r"(pA), "=r"(mB), "=r"(pB)
                                     : "r"(rmh + (b * (kReplayRows / 2) + r / 2) * 16)
                                     : "memory");
                        if ((mA >> lane) & 1u) __stcg(out_tile + (pA + __popc(mA & lt)), idx);
                        if ((mB >> lane) & 1u) __stcg(out_tile + (pB + __popc(mB & lt)), idx);
                    }
                };
                while (nz) {
                    const int b1 = 31 - __clz(nz);  // order is free: every buffer's start is known
                    nz ^= 1u << b1;
                    if (nz) {
                        const int b2 = 31 - __clz(nz);
                        nz ^= 1u << b2;
                        step(b1);
                        step(b2);
                    } else {
                        step(b1);
                    }
                }
            }
            cursor += adv;
        }
    }
}

// Max records per tile for the fused count -> replay fill (128 buffers x 256 B = 32 KB).
constexpr u32 kRecCap = 128;
// LO_REC_CAP (test knob, read per call): a smaller per-tile record cap forces the overflow path
inline u32 rec_cap() {
    const char* e = std::getenv("LO_REC_CAP");
    const unsigned long v = e ? std::strtoul(e, nullptr, 10) : 0;
    return v >= 1 && v <= kRecCap ? static_cast<u32>(v) : kRecCap;
}

// The count pass's record pool in the persistent context arena: rec_off[tiles] u64 | alloc u64 |
// rec_n[tiles] | overflow list[tiles] | ovf_n | pool (records of 256 B).  The pool is sized for
// the worst case (cap per tile) within a quarter of the free memory; tiles that find it
// exhausted fall back to the fill walk.  Throws LO_OUT_OF_MEMORY when even that cannot be had.
struct RecSetup {
    RecPool rp;
    u32* ovf = nullptr;
    u32* ovf_n = nullptr;
};
static inline RecSetup setup_records(lo_context* ctx, u64 tiles, u32 cap) {
    SlowLog slow("setup_records", tiles);
    RecSetup rs;
    const u64 head = 8 * (tiles + 1) + 4 * (2 * tiles + 1);
    u64 recs = tiles * cap;
    const u64 demand = head + 16 + recs * 256;
    // cudaMemGetInfo is queried only when the demand outgrows what the arena was last budgeted for:
    // it blocked the host for 2-70 ms at random while the GPU was busy, idling the device mid-step
    const bool reuse = demand <= ctx->arena_bytes ||
                       (demand <= ctx->arena_budgeted && ctx->arena_bytes >= head + 16 + 2 * kRecChunk * 256);
    if (reuse) {  // whatever the arena holds
        recs = (ctx->arena_bytes - head - 16) / 256;
    } else {  // growing: respect free memory
        size_t free_b = 0, total_b = 0;
        LO_CUDA(cudaMemGetInfo(&free_b, &total_b));
        const u64 budget = (free_b + ctx->arena_bytes) / 4;
        recs = std::min<u64>(recs, budget > head ? (budget - head) / 256 : 0);
        ctx->arena_budgeted = demand;
    }
    recs = std::max<u64>(recs, kRecChunk * 2);
    unsigned char* base = static_cast<unsigned char*>(arena(ctx, head + 16 + recs * 256));
    rs.rp.rec_off = reinterpret_cast<u64*>(base);
    rs.rp.alloc = rs.rp.rec_off + tiles;
    rs.rp.rec_n = reinterpret_cast<u32*>(rs.rp.alloc + 1);
    rs.ovf = rs.rp.rec_n + tiles;
    rs.ovf_n = rs.ovf + tiles;
    rs.rp.pool = reinterpret_cast<u32*>(base + ((head + 15) / 16) * 16);
    rs.rp.pool_recs = recs;
    rs.rp.cap = cap;
    LO_CUDA(cudaMemsetAsync(rs.rp.alloc, 0, 8, ctx->stream));
    return rs;
}

// Diagnostic (LO_REPLAY_STATS): the records' shape -- records per tile, (row, record) pairs with
// members, and the sum over records of the largest per-row member count -- printed to stderr.
static inline void replay_stats(lo_context* ctx, const RecSetup& rs, u64 m, u64 tiles) {
    std::vector<u32> rn(tiles);
    std::vector<u64> ro(tiles);
    u64 alloc = 0;
    LO_CUDA(cudaMemcpyAsync(rn.data(), rs.rp.rec_n, 4 * tiles, cudaMemcpyDeviceToHost, ctx->stream));
    LO_CUDA(cudaMemcpyAsync(ro.data(), rs.rp.rec_off, 8 * tiles, cudaMemcpyDeviceToHost, ctx->stream));
    LO_CUDA(cudaMemcpyAsync(&alloc, rs.rp.alloc, 8, cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    alloc = std::min<u64>(alloc, rs.rp.pool_recs);
    std::vector<u32> pool(alloc * 64);
    LO_CUDA(cudaMemcpyAsync(pool.data(), rs.rp.pool, 256 * alloc, cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    double recs = 0, pairs = 0, maxsum = 0, members = 0, used = 0;
    u64 hist[9] = {};
    for (u64 t = 0; t < tiles; ++t) {
        if (rn[t] == kRecOverflow) continue;
        used += 1;
        recs += rn[t];
        hist[std::min<u32>(8, rn[t] / 16)]++;
        for (u32 b = 0; b < rn[t]; ++b) {
            const u32* R = pool.data() + (ro[t] + b) * 64;
            u32 mx = 0;
            for (u32 L = 0; L < 32; ++L) {
                const u32 c = static_cast<u32>(__builtin_popcount(R[32 + L]));
                pairs += c != 0;
                members += c;
                mx = std::max(mx, c);
            }
            maxsum += mx;
        }
    }
    std::fprintf(stderr,
                 "[lo] replay stats: m=%llu tiles=%llu recorded=%.0f recs/tile=%.1f pairs/tile=%.1f "
                 "members/tile=%.1f members/pair=%.2f maxpop-sum/tile=%.1f  n-hist(16s):",
                 static_cast<unsigned long long>(m), static_cast<unsigned long long>(tiles), used, recs / used,
                 pairs / used, members / used, members / std::max(1.0, pairs), maxsum / used);
    for (u64 h : hist) std::fprintf(stderr, " %llu", static_cast<unsigned long long>(h));
    std::fprintf(stderr, "\n");
}

// Fill by replaying the records into the CSR (offsets[m+1], out); returns how many tiles
// overflowed (their ids in rs.ovf) and need the fill walk.
static inline u32 replay_records(lo_context* ctx, const RecSetup& rs, u64 m, const u64* offsets, u32* out,
                                 u64 total) {
    const u64 tiles = (m + 31) / 32;
    LO_CUDA(cudaMemsetAsync(rs.ovf_n, 0, 4, ctx->stream));
    // short rows: buffer-major stores stay line-local; long rows: row-major so every output line
    // completes while hot (measured crossover ~ 32-45 members per row: cfg1 r = 1 (31.5) is faster
    // buffer-major, cfg4 (45) and cfg0 (65) row-major)
    static const u64 row_major_min = [] {
        const char* e = std::getenv("LO_REPLAY_ROW_MAJOR_MIN");
        return e ? std::strtoull(e, nullptr, 10) : 40ull;
    }();
    if (total < row_major_min * m) {
        const int rb = static_cast<int>(std::max<u64>(
            1, std::min<u64>((tiles + kReplayWarps - 1) / kReplayWarps, ctx->sm_count * 16ull)));
        radius_replay_bm_kernel<<<rb, 128, 0, ctx->stream>>>(rs.rp, m, offsets, out, rs.ovf, rs.ovf_n);
    } else {
        ensure_smem_attr(ctx, kAttrReplay, radius_replay_kernel, kReplaySmem);
        const int rr = static_cast<int>(std::max<u64>(
            1, std::min<u64>((tiles + kReplayWarps - 1) / kReplayWarps, ctx->sm_count * static_cast<u64>(kReplayBlocks))));
        radius_replay_kernel<<<rr, 32 * kReplayWarps, kReplaySmem, ctx->stream>>>(rs.rp, m, offsets, out, rs.ovf,
                                                                                rs.ovf_n);
    }
    LO_CHECK_LAUNCH();
    static const bool stats = std::getenv("LO_REPLAY_STATS") != nullptr;
    if (stats) replay_stats(ctx, rs, m, tiles);
    return read_scalar(ctx, rs.ovf_n);
}

// Point tests relative to a tile origin.  The FP32 filter's error bound grows with the magnitude
// of the FP32 coordinates (search_common.cuh: d = 2 * 2^-23 * B + 2^-23 * 2r, B >= |p - o|).
// Relative to the cloud origin B is the cube side (~3 km at cfg3, d ~ 7e-4 at r = 1, so ~1 % of
// the candidate pairs fell in the FP64 band); relative to the tile's first query, B only has to
// bound |p - o_t| for candidates that can be near the threshold, i.e. within 2r of a tile query:
// B = max_tile |q - o_t| + 2r, a few metres.  Farther candidates are outside whatever their
// rounding: their FP32 difference keeps its relative error <= 2^-23 and exceeds 1.99 r on some
// axis (d < 0.01 r).  Candidate and query coordinates are rounded from FP64 differences
// fl32(fl64(p - o_t)), exactly the model of the bound.  A tile too wide for the test
// (d >= 0.01 r) sends every candidate to the exact predicate (lo = 0, hi = +inf).
struct TileTest {
    float lo, hi;  // Sphere / Circle: squared-distance thresholds; Cube / Square: L-inf ones
};
template <int SHAPE>
__device__ __forceinline__ TileTest tile_test(double r, double ext) {
    const double u = 0x1p-23;
    const double B = ext + 2.0 * r;
    const double d = 2.0 * u * B + u * 2.0 * r;
    const double r2 = r * r;
    TileTest t;
    if (!(d < 0.01 * r)) {
        t.lo = 0.f;
        t.hi = INFINITY;
        return t;
    }
    if (SHAPE == LO_SPHERE || SHAPE == LO_CIRCLE) {
        const double M = 1.25 * (3.0 * u * 4.0 * r2 + 2.0 * 1.7320508075688772 * 2.0 * r * d + 3.0 * d * d +
                                 0x1p-49 * 4.0 * r2);
        t.lo = __double2float_rd(r2 - M);
        t.hi = __double2float_ru(r2 + M);
    } else {
        const double ml = 1.25 * (d + 0x1p-50 * r);
        t.lo = __double2float_rd(r - ml);
        t.hi = __double2float_ru(r + ml);
    }
    return t;
}

// DIGEST (count pass only): the FNV-1a-64 row digests (search.cpp:263-271, :345-347) are folded in
// as the members are found -- buffers follow the DFS code order and slots keep point order, so
// lane L meets row L's members in ascending order, exactly the order the digest hashes them.
// This replaces a separate pass that re-read every CSR row (25.5 GB at cfg3).  1: u32 indices,
// 2: indices < 2^24 (five zero bytes fold into one multiply).
template <int SHAPE, bool FILL, int DIGEST = 0>
__global__ void __launch_bounds__(kPtThreads, LO_PT_MINB) radius_pt_kernel(
    const TNodeF* __restrict__ tf, const float4* __restrict__ pf, const double* __restrict__ px,
    const double* __restrict__ py, const double* __restrict__ pz, Queries q, FloatTest ft,
    float compact, double r, double r2, u32* __restrict__ counts, const u64* __restrict__ offsets,
    u32* __restrict__ out, u64* tile_counter, RecPool rp, const u32* __restrict__ tile_list,
    u64 list_n, u64* __restrict__ fps) {
    __shared__ PtShared shared_s[kPtWarps];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    PtShared& S = shared_s[w];
    const u64 ntiles = tile_list ? list_n : (q.m + 31) / 32;
    const int cl = lane & 7, grp = lane >> 3;
    u64 chunk_base = 0;  // count pass: this warp's current record chunk (in records)
    u32 chunk_left = 0;
    for (;;) {
        u64 tile = 0;
        if (lane == 0) tile = atomicAdd(reinterpret_cast<unsigned long long*>(tile_counter), 1ull);
        tile = __shfl_sync(~0u, tile, 0);
        if (tile >= ntiles) break;
        if (tile_list) tile = tile_list[tile];  // fill fallback for tiles the records missed
        if (!FILL && rp.pool && chunk_left < rp.cap) {
            // a fresh chunk so this tile's records stay contiguous
            u64 base = 0;
            if (lane == 0) base = atomicAdd(reinterpret_cast<unsigned long long*>(rp.alloc),
                                            static_cast<unsigned long long>(kRecChunk));
            base = __shfl_sync(~0u, base, 0);
            chunk_base = base;
            chunk_left = base + kRecChunk <= rp.pool_recs ? kRecChunk : 0u;
        }
        const u64 qi = tile * 32 + lane;
        const bool active = qi < q.m;
        double cx = 0.0, cy = 0.0, cz = 0.0;
        float4 qf = make_float4(INFINITY, INFINITY, INFINITY, 0.f);  // never near anything
        if (active) {
            load_query(q, qi, cx, cy, cz);
            qf = load_query_f(q, qi);
        }
        // tile origin = the tile's first query (lane 0 is active in every tile)
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
            S.qx[lane] = S.qy[lane] = S.qz[lane] = INFINITY;  // never near anything
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ext = fmaxf(ext, __shfl_xor_sync(~0u, ext, o));
        const TileTest tt = tile_test<SHAPE>(r, static_cast<double>(ext));
        const float lo_thr = tt.lo, hi_thr = tt.hi;
        S.qd[lane][0] = cx;
        S.qd[lane][1] = cy;
        S.qd[lane][2] = cz;
        // fill: rows of the tile are contiguous from offsets[tile*32]; cursors are relative
        u32* out_tile = out;
        u32 mine = 0;
        if (FILL) {
            const u64 tbase = offsets[tile * 32];
            out_tile = out + tbase;
            mine = active ? static_cast<u32>(offsets[qi] - tbase) : 0u;
        }
        float gl[3] = {qf.x, qf.y, qf.z}, gh[3] = {qf.x, qf.y, qf.z};
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                gl[a] = fminf(gl[a], __shfl_xor_sync(~0u, gl[a], o));
                gh[a] = fmaxf(gh[a], __shfl_xor_sync(~0u, gh[a], o));
            }
        }
        const bool gcompact = fmaxf(fmaxf(gh[0] - gl[0], gh[1] - gl[1]), gh[2] - gl[2]) <= compact;
        // the whole tile's query box: candidate points farther than r from it are members of no
        // query of the tile (tile_disjoint_f with the point as a degenerate box), so they are
        // dropped before they take a buffer slot
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            float tl = fminf(gl[a], __shfl_xor_sync(~0u, gl[a], 8));
            float th = fmaxf(gh[a], __shfl_xor_sync(~0u, gh[a], 8));
            tl = fminf(tl, __shfl_xor_sync(~0u, tl, 16));
            th = fmaxf(th, __shfl_xor_sync(~0u, th, 16));
            if (lane == 0) S.tbox[a] = tl, S.tbox[3 + a] = th;
        }
        u32 fill = 0, qmask = 0;  // buffer occupancy and interested queries (warp-uniform)
        u32 nrec = 0;             // count pass: buffers recorded for the replay
        u64 hash = kFnvOffset;    // DIGEST: row L's FNV-1a-64 so far
        u32* rec_tile = (!FILL && rp.pool && chunk_left >= rp.cap) ? rp.pool + chunk_base * 64 : nullptr;
        auto flush = [&]() {
            // the buffer's points are loaded here, all 32 at once (one latency per buffer instead
            // of one per leaf); slots >= fill get +INF coordinates, never members
            float4 P = make_float4(INFINITY, INFINITY, INFINITY, 0.f);
            if (static_cast<u32>(lane) < fill) {
                const u32 g = S.bix[lane];
                // tile origin = query 0, re-read from shared memory (registers are the limit)
                P = make_float4(__double2float_rn(__ldg(px + g) - S.qd[0][0]),
                                __double2float_rn(__ldg(py + g) - S.qd[0][1]),
                                __double2float_rn(__ldg(pz + g) - S.qd[0][2]), __uint_as_float(g));
            }
            u32 mymask = 0;
            process_buffer<SHAPE, FILL>(S, P, fill, qmask, lane, lo_thr, hi_thr, px, py, pz, r, r2,
                                        out_tile, mine, mymask);
            if (!FILL) {
                mine += __popc(mymask);
                if (DIGEST) {
                    for (u32 mm = mymask; mm; mm &= mm - 1) {
                        const u32 g = S.bix[__ffs(mm) - 1];
                        hash = DIGEST == 2 ? fnv_u24(hash, g) : fnv_u32(hash, g);
                    }
                }
                // buffers without members leave no record (the replay would skip them anyway)
                if (rec_tile && __any_sync(~0u, mymask != 0)) {
                    if (nrec < rp.cap) {
                        u32* R = rec_tile + nrec * 64;
                        R[lane] = __float_as_uint(P.w);
                        R[32 + lane] = mymask;
                    }
                    ++nrec;
                }
            }
        };
#if LO_PT_STREAM
        // The walk queues the leaves it keeps (up to 32); drain() streams their points 32 at a time
        // across leaf boundaries -- lane j takes stream position s0 + j, its leaf found by a popcount
        // over the leaves' start positions -- with the next 32 points' loads in flight while the
        // current ones are filtered against the tile box and appended to the buffer.
        u32 nl = 0;
        auto drain = [&]() {
            __syncwarp();
            const u32 sz = static_cast<u32>(lane) < nl ? S.lsize[lane] : 0u;
            u32 inc = sz;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const u32 t = __shfl_up_sync(~0u, inc, o);
                if (lane >= o) inc += t;
            }
            const u32 total = __shfl_sync(~0u, inc, 31);
            // leaf `lane`'s stream start replaces its size; the rest of the lookup goes through
            // shared memory (registers are the kernel's limit)
            const u32 lst = static_cast<u32>(lane) < nl && sz != 0 ? inc - sz : 0xffffffffu;
            if (static_cast<u32>(lane) < nl) S.lsize[lane] = inc - sz;
            __syncwarp();
            const u32 le = (2u << lane) - 1u;  // lanes <= this one (lane 31: all)
            // point of stream position s0 + lane: index and leaf slot (valid only below total)
            auto locate = [&](u32 s0, u32& g, u32& j) {
                const u32 before = __popc(__ballot_sync(~0u, lst < s0));
                const u32 rel = lst - s0;
                const u32 B = __reduce_or_sync(~0u, lst != 0xffffffffu && lst >= s0 && rel < 32u ? 1u << rel : 0u);
                j = (before + __popc(B & le) - 1u) & 31u;
                g = S.lbeg[j] + (s0 + static_cast<u32>(lane) - S.lsize[j]);
            };
            // the next 32 points travel by cp.async straight into this warp's shared slots, so no
            // registers are held across the buffer flushes
            u32 g, j;
            locate(0, g, j);
            bool valid = static_cast<u32>(lane) < total;
            const u32 pre0 = static_cast<u32>(__cvta_generic_to_shared(&S.pre[0][lane]));
            if (valid) asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(pre0), "l"(pf + g) : "memory");
            asm volatile("cp.async.commit_group;" ::: "memory");
            u32 ph = 0;
            for (u32 s0 = 0; s0 < total; s0 += 32, ph ^= 1u) {
                u32 g2 = 0, j2 = 0;
                const bool valid2 = s0 + 32 + static_cast<u32>(lane) < total;
                if (s0 + 32 < total) {
                    locate(s0 + 32, g2, j2);
                    if (valid2)
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(pre0 + (ph ^ 1u) * 512u),
                                     "l"(pf + g2)
                                     : "memory");
                    asm volatile("cp.async.commit_group;" ::: "memory");
                    asm volatile("cp.async.wait_group 1;" ::: "memory");
                } else {
                    asm volatile("cp.async.wait_group 0;" ::: "memory");
                }
                float3 cur = make_float3(0.f, 0.f, 0.f);
                if (valid) {
                    const float4 c4 = S.pre[ph][lane];
                    cur = make_float3(c4.x, c4.y, c4.z);
                }
                bool ok = false;
                if (valid) {
                    NodeF pt;
                    pt.lo[0] = pt.hi[0] = cur.x;
                    pt.lo[1] = pt.hi[1] = cur.y;
                    pt.lo[2] = pt.hi[2] = cur.z;
                    ok = !tile_disjoint_f<SHAPE>(S.tbox, S.tbox + 3, pt, ft);
                }
                const u32 bal = __ballot_sync(~0u, ok);
                if (bal) {
                    const u32 wv = ok ? S.lwant[j] : 0u;
                    const u32 pos = fill + __popc(bal & ((1u << lane) - 1u));
                    __syncwarp();
                    if (ok && pos < 32) S.bix[pos] = g;
                    qmask |= __reduce_or_sync(~0u, pos < 32 ? wv : 0u);
                    fill += __popc(bal);
                    if (fill >= 32) {
                        const u32 over = fill - 32;
                        fill = 32;
                        __syncwarp();
                        flush();
                        __syncwarp();
                        if (ok && pos >= 32) S.bix[pos - 32] = g;
                        fill = over;
                        qmask = __reduce_or_sync(~0u, pos >= 32 ? wv : 0u);
                    }
                }
                g = g2, j = j2, valid = valid2;
            }
            nl = 0;
            __syncwarp();
        };
#endif
        int sp = 1;
        if (lane == 0) S.stack[0] = 0;
        __syncwarp();
        while (sp > 0) {
            const u32 t = S.stack[--sp];
            const NodeF nd = load_node_f(tf, t);
            if (nd.nchild != 0 && nd.end - nd.begin > ft.coarse) {
                bool keep = false;
                if (cl < static_cast<int>(nd.nchild)) {
                    const NodeF ch = load_node_f(tf, nd.child0 + cl);
                    if (gcompact) {
                        keep = !tile_disjoint_f<SHAPE>(gl, gh, ch, ft);
                    } else {
#pragma unroll
                        for (int j = 0; j < 8; ++j) keep |= !disjoint_f<SHAPE>(S.qf[8 * grp + j], ch, ft);
                    }
                }
                u32 s = __ballot_sync(~0u, keep);
                s = (s | (s >> 8) | (s >> 16) | (s >> 24)) & 0xffu;
                const int k = __popc(s);
                __syncwarp();
                if (lane < 8 && ((s >> lane) & 1u))
                    S.stack[sp + k - 1 - __popc(s & ((1u << lane) - 1u))] = nd.child0 + lane;
                sp += k;
                __syncwarp();
                continue;
            }
            // leaf: which queries can reach it
            const u32 want = __ballot_sync(~0u, active && !disjoint_f<SHAPE>(qf, nd, ft));
            if (!want) continue;
#if LO_PT_STREAM
            if (lane == 0) {
                S.lbeg[nl] = nd.begin;
                S.lsize[nl] = nd.end - nd.begin;
                S.lwant[nl] = want;
            }
            if (++nl == 32) drain();
            continue;
#endif
#if LO_PT_PREFILTER
            for (u32 b0 = nd.begin; b0 < nd.end; b0 += 32) {
                const u32 g = b0 + static_cast<u32>(lane);
                bool ok = false;
                if (g < nd.end) {
                    const float4 pp = __ldg(pf + g);
                    NodeF pt;
                    pt.lo[0] = pt.hi[0] = pp.x;
                    pt.lo[1] = pt.hi[1] = pp.y;
                    pt.lo[2] = pt.hi[2] = pp.z;
                    ok = !tile_disjoint_f<SHAPE>(S.tbox, S.tbox + 3, pt, ft);
                }
                const u32 bal = __ballot_sync(~0u, ok);
                if (!bal) continue;
                const u32 pos = fill + __popc(bal & ((1u << lane) - 1u));
                __syncwarp();
                if (ok && pos < 32) S.bix[pos] = g;
                fill += __popc(bal);
                qmask |= want;
                if (fill >= 32) {
                    const u32 over = fill - 32;
                    fill = 32;
                    __syncwarp();
                    flush();
                    __syncwarp();
                    if (ok && pos >= 32) S.bix[pos - 32] = g;
                    fill = over;
                    qmask = over ? want : 0u;
                }
            }
#else
            for (u32 base = nd.begin; base < nd.end;) {
                const u32 take = min(32u - fill, nd.end - base);
                __syncwarp();
                if (static_cast<u32>(lane) < take) S.bix[fill + lane] = base + lane;
                fill += take;
                qmask |= want;
                base += take;
                if (fill == 32) {
                    __syncwarp();
                    flush();
                    fill = 0;
                    qmask = 0;
                }
            }
#endif
        }
#if LO_PT_STREAM
        if (nl) drain();
#endif
        if (fill) {
            __syncwarp();
            flush();  // partial last buffer
        }
        if (!FILL && active) counts[qi] = mine;
        if (DIGEST && active) fps[qi] = hash;
        if (!FILL && rp.pool) {
            const bool ok = rec_tile && nrec <= rp.cap;
            if (lane == 0) {
                rp.rec_n[tile] = ok ? nrec : kRecOverflow;
                rp.rec_off[tile] = chunk_base;
            }
            if (ok) {
                chunk_base += nrec;
                chunk_left -= nrec;
            }
        }
        __syncwarp();
    }
}

}  // namespace lo
