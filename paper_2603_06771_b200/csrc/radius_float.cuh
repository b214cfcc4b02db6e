// radius_float.cuh -- the FP32-filtered radius walk (K6 count / fill), included by radius.cu.
//
// One warp = 32 consecutive queries.  Internal nodes: lane (child c, query group g) tests
// child c against group g's 8 queries -- by their FP32 bounding box when the group is compact,
// one by one otherwise -- so a child is entered only if some query may reach it.  Leaves: each
// lane classifies the leaf box (Contains -> whole range, Disjoint -> skip), then the leaf's
// points are staged in shared memory as (x0,x1,y0,y1 | z0,z1) pairs and tested two at a time
// with packed FP32 math (FADD2 / FMUL2 / FFMA2 on sm_100a) against the rigorous thresholds of
// search_common.cuh; the rare points in the uncertainty band are decided by the exact FP64
// predicate.  Rows come out ascending because children are visited in code order.
#pragma once

#include "search_common.cuh"

namespace lo {

__device__ __forceinline__ u64 pack2(float a, float b) {
    u64 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void unpack2(u64 v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ u64 fsub2(u64 a, u64 b) {
    u64 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ u64 fmul2(u64 a, u64 b) {
    u64 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) {
    u64 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

constexpr int kRadiusWarps = 4;
constexpr int kRadiusThreads = 32 * kRadiusWarps;

// Fill-pass write combining: each lane stages its row in a 64-slot shared-memory ring (row
// stride 65 words, so a flush reads 32 consecutive slots of one lane conflict-free); as soon
// as a lane has 32 staged indices the warp stores them as one coalesced 128-byte run instead
// of 32 scattered 4-byte stores.  A chunk adds at most 32, so 64 slots never overflow.
constexpr u32 kRing = 64;
constexpr u32 kRingStride = kRing + 1;

__device__ __forceinline__ void ring_append(u32* ring, int lane, u32& rs, u32& rn, u32 in,
                                            u32 base, u64& rowpos, u32* __restrict__ out) {
    u32* mine = ring + lane * kRingStride;
    while (in) {
        const int b = __ffs(in) - 1;
        in &= in - 1;
        mine[(rs + rn) & (kRing - 1)] = base + b;
        ++rn;
    }
    __syncwarp();
    unsigned fm = __ballot_sync(~0u, rn >= 32);
    while (fm) {
        const int L = __ffs(fm) - 1;
        fm &= fm - 1;
        const u32 sL = __shfl_sync(~0u, rs, L);
        const u64 pL = __shfl_sync(~0u, rowpos, L);
        out[pL + lane] = ring[L * kRingStride + ((sL + lane) & (kRing - 1))];
    }
    __syncwarp();
    if (rn >= 32) {
        rs = (rs + 32) & (kRing - 1);
        rn -= 32;
        rowpos += 32;
    }
}

template <int SHAPE, bool FILL>
__global__ void __launch_bounds__(kRadiusThreads, 8) radius_float_kernel(
    const TNodeF* __restrict__ tf, const float4* __restrict__ pf, const double* __restrict__ px,
    const double* __restrict__ py, const double* __restrict__ pz, Queries q, FloatTest ft,
    float compact, double r, double r2, u32* __restrict__ counts, const u64* __restrict__ offsets,
    u32* __restrict__ out, u64* tile_counter) {
    __shared__ u32 stack_s[kRadiusWarps][kStackCap];
    __shared__ float4 pa_s[kRadiusWarps][16];  // (x0, x1, y0, y1) per candidate pair
    __shared__ float2 pb_s[kRadiusWarps][16];  // (z0, z1)
    __shared__ float4 sq_s[kRadiusWarps][32];
    __shared__ u32 ring_s[FILL ? kRadiusWarps : 1][FILL ? 32 * kRingStride : 1];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    u32* ring = ring_s[FILL ? w : 0];
    u32* stack = stack_s[w];
    float4* pa = pa_s[w];
    float2* pb = pb_s[w];
    float* paf = reinterpret_cast<float*>(pa);
    float* pbf = reinterpret_cast<float*>(pb);
    float4* squeries = sq_s[w];
    const u64 ntiles = (q.m + 31) / 32;
    const int cl = lane & 7, grp = lane >> 3;
    constexpr bool kPacked = SHAPE == LO_SPHERE || SHAPE == LO_CIRCLE;
    const float lo_thr = kPacked ? ft.t_lo : ft.r_lo;
    const float hi_thr = kPacked ? ft.t_hi : ft.r_hi;
    for (;;) {
        // dynamic tile scheduling: heavy tiles (dense clusters) do not stall a static stride
        u64 tile = 0;
        if (lane == 0) tile = atomicAdd(reinterpret_cast<unsigned long long*>(tile_counter), 1ull);
        tile = __shfl_sync(~0u, tile, 0);
        if (tile >= ntiles) break;
        const u64 qi = tile * 32 + lane;
        const bool active = qi < q.m;
        double cx = 0.0, cy = 0.0, cz = 0.0;
        float4 qf = make_float4(INFINITY, INFINITY, INFINITY, 0.f);  // never near anything
        if (active) {
            load_query(q, qi, cx, cy, cz);
            qf = load_query_f(q, qi);
        }
        __syncwarp();
        squeries[lane] = qf;
        // the box of this lane's 8-query group, and whether it is compact enough to stand in
        // for the 8 queries in child tests (a pruned child is disjoint for all of them)
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
        const u64 QX = pack2(qf.x, qf.x), QY = pack2(qf.y, qf.y), QZ = pack2(qf.z, qf.z);
        u32 count = 0;
        u64 rowpos = 0;  // CSR position of this lane's next flushed index (fill pass)
        u32 rs = 0, rn = 0;  // ring start slot / staged count of this lane (fill pass)
        if (FILL && active) rowpos = offsets[qi];
        int sp = 1;
        if (lane == 0) stack[0] = 0;
        __syncwarp();
        while (sp > 0) {
            const u32 t = stack[--sp];
            const NodeF nd = load_node_f(tf, t);
            if (nd.nchild != 0) {
                bool keep = false;
                if (cl < static_cast<int>(nd.nchild)) {
                    const NodeF ch = load_node_f(tf, nd.child0 + cl);
                    if (gcompact) {
                        keep = !tile_disjoint_f<SHAPE>(gl, gh, ch, ft);
                    } else {
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            keep |= !disjoint_f<SHAPE>(squeries[8 * grp + j], ch, ft);
                    }
                }
                u32 s = __ballot_sync(~0u, keep);
                s = (s | (s >> 8) | (s >> 16) | (s >> 24)) & 0xffu;
                const int k = __popc(s);
                __syncwarp();
                if (lane < 8 && ((s >> lane) & 1u))
                    stack[sp + k - 1 - __popc(s & ((1u << lane) - 1u))] = nd.child0 + lane;
                sp += k;
                __syncwarp();
                continue;
            }
            int rel = kDisjoint;
            if (active) rel = relation_f<SHAPE>(qf, nd, ft);
            // lanes whose query contains the whole leaf take its range without point tests
            // (neighbours_prune's Contains shortcut)
            const bool any_isect = __any_sync(~0u, rel == kIntersects);
            if (!any_isect && !__any_sync(~0u, rel == kContains)) continue;
            for (u32 base = nd.begin; base < nd.end; base += 32) {
                const u32 cnt = min(32u, nd.end - base);
                if (!any_isect) {
                    // only Contains lanes: whole chunks, no staging
                    const u32 in = rel == kContains ? (cnt == 32 ? ~0u : ((1u << cnt) - 1u)) : 0u;
                    if (FILL) ring_append(ring, lane, rs, rn, in, base, rowpos, out);
                    count += __popc(in);
                    continue;
                }
                __syncwarp();
                if (static_cast<u32>(lane) < cnt) {
                    const float4 p = __ldg(pf + base + lane);
                    const int pp = lane >> 1, h = lane & 1;
                    paf[4 * pp + h] = p.x;
                    paf[4 * pp + 2 + h] = p.y;
                    pbf[2 * pp + h] = p.z;
                }
                __syncwarp();
                u32 in = 0, band = 0;
                if (rel == kIntersects) {
                    const u32 npairs = (cnt + 1) >> 1;
                    for (u32 pp = 0; pp < npairs; ++pp) {
                        const float4 a = pa[pp];
                        float v0, v1;
                        if (kPacked) {
                            const u64 dx = fsub2(pack2(a.x, a.y), QX);
                            const u64 dy = fsub2(pack2(a.z, a.w), QY);
                            u64 d2 = fmul2(dx, dx);
                            d2 = ffma2(dy, dy, d2);
                            if (SHAPE == LO_SPHERE) {
                                const float2 b = pb[pp];
                                const u64 dz = fsub2(pack2(b.x, b.y), QZ);
                                d2 = ffma2(dz, dz, d2);
                            }
                            unpack2(d2, v0, v1);
                        } else {
                            const float2 b = pb[pp];
                            v0 = metric_f<SHAPE>(qf, make_float4(a.x, a.z, b.x, 0.f));
                            v1 = metric_f<SHAPE>(qf, make_float4(a.y, a.w, b.y, 0.f));
                        }
                        const u32 bit = 1u << (2 * pp);
                        if (v0 < lo_thr) in |= bit;
                        if (v0 < hi_thr) band |= bit;
                        if (v1 < lo_thr) in |= bit << 1;
                        if (v1 < hi_thr) band |= bit << 1;
                    }
                    const u32 valid = cnt == 32 ? ~0u : ((1u << cnt) - 1u);
                    in &= valid;
                    band &= valid & ~in;
                    while (band) {  // rare: the exact FP64 predicate decides
                        const int b = __ffs(band) - 1;
                        band &= band - 1;
                        const u32 g = base + b;
                        if (contains<SHAPE>(cx, cy, cz, r, r2, px[g], py[g], pz[g])) in |= 1u << b;
                    }
                } else if (rel == kContains) {
                    in = cnt == 32 ? ~0u : ((1u << cnt) - 1u);
                }
                if (FILL) ring_append(ring, lane, rs, rn, in, base, rowpos, out);
                count += __popc(in);
            }
        }
        if (FILL) {
            // drain: every lane's remaining (< 64) staged indices
            unsigned fm = __ballot_sync(~0u, rn > 0);
            while (fm) {
                const int L = __ffs(fm) - 1;
                fm &= fm - 1;
                const u32 nL = __shfl_sync(~0u, rn, L);
                const u32 sL = __shfl_sync(~0u, rs, L);
                const u64 pL = __shfl_sync(~0u, rowpos, L);
                for (u32 i = lane; i < nL; i += 32) out[pL + i] = ring[L * kRingStride + ((sL + i) & (kRing - 1))];
            }
            __syncwarp();
            rn = 0;
            rs = 0;
        }
        if (!FILL && active) counts[qi] = count;
        __syncwarp();
    }
}

}  // namespace lo
