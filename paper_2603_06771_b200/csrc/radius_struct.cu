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

#include "radius_pt.cuh"

namespace lo {

// ---- fast path: the lin count kernel's lane = point buffers + the FP32 filter ----------------
// Node relations against the reference's octant boxes are decided in FP32 on outward-rounded
// copies of those boxes (rbf) with the FloatTest margins -- Contains iff far^2 < t_lo, not
// Contains iff far^2 >= t_hi, Disjoint iff near^2 >= t_hi, not Disjoint iff near^2 < t_lo -- and
// only the band in between is evaluated in FP64 on the exact boxes (rb).  Leaf points go through
// the 32-slot buffers; each slot carries the mask of queries that reached its leaf as Intersects,
// so a query that contains (or skipped) that leaf never counts its points as singles.
enum { kRelU = 3 };  // "uncertain": decide in FP64
constexpr u32 kStructRangeCap = 16;  // count-pass range slots per query (more: the tile is re-walked)

// Ranges of the count pass (per query scratch) into the ranges CSR; overflowed tiles are written
// by the fill walk instead.
__global__ void struct_copy_ranges(const u32* __restrict__ rscratch, const u32* __restrict__ nrng, u64 m,
                                   const u64* __restrict__ r_off, const u32* __restrict__ rec_n,
                                   u32* __restrict__ ranges) {
    for (u64 e = blockIdx.x * (u64)blockDim.x + threadIdx.x; e < m * kStructRangeCap;
         e += (u64)gridDim.x * blockDim.x) {
        const u64 qi = e / kStructRangeCap, j = e - qi * kStructRangeCap;
        if (j >= nrng[qi] || rec_n[qi / 32] == kRecOverflow) continue;
        const uint2 v = reinterpret_cast<const uint2*>(rscratch)[e];
        reinterpret_cast<uint2*>(ranges)[r_off[qi] + j] = v;
    }
}

template <int SHAPE>
__device__ __forceinline__ int classify_ref_f(const float4& q, const float4& lo, const float4& hi,
                                              const FloatTest& ft) {
    const float nx = fmaxf(fmaxf(lo.x - q.x, q.x - hi.x), 0.f);
    const float ny = fmaxf(fmaxf(lo.y - q.y, q.y - hi.y), 0.f);
    const float fx = fmaxf(q.x - lo.x, hi.x - q.x);
    const float fy = fmaxf(q.y - lo.y, hi.y - q.y);
    float nm, fm, tl, th;
    if (SHAPE == LO_SPHERE || SHAPE == LO_CUBE) {
        const float nz = fmaxf(fmaxf(lo.z - q.z, q.z - hi.z), 0.f);
        const float fz = fmaxf(q.z - lo.z, hi.z - q.z);
        if (SHAPE == LO_SPHERE) {
            nm = fmaf(nz, nz, fmaf(ny, ny, nx * nx));
            fm = fmaf(fz, fz, fmaf(fy, fy, fx * fx));
            tl = ft.t_lo, th = ft.t_hi;
        } else {
            nm = fmaxf(fmaxf(nx, ny), nz);
            fm = fmaxf(fmaxf(fx, fy), fz);
            tl = ft.r_lo, th = ft.r_hi;
        }
    } else if (SHAPE == LO_CIRCLE) {
        nm = fmaf(ny, ny, nx * nx);
        fm = fmaf(fy, fy, fx * fx);
        tl = ft.t_lo, th = ft.t_hi;
    } else {
        nm = fmaxf(nx, ny);
        fm = fmaxf(fx, fy);
        tl = ft.r_lo, th = ft.r_hi;
    }
    if (fm < tl) return kContains;
    if (fm < th) return kRelU;
    if (nm >= th) return kDisjoint;
    if (nm >= tl) return kRelU;
    return kIntersects;
}

struct StructShared {
    PtShared pt;
    u32 sw[32];  // per buffer slot: queries that reached the slot's leaf as Intersects
};

// Tests the buffer (lane j = slot j) against every query whose bit is in qmask; a query counts a
// slot only if the slot's want mask holds it.  Count pass (records): query L's membership mask of
// the buffer lands in S.msk[L] (quads of queries per ballot round for the packed shapes).  Fill
// walk: members of query L go to singles[srow_L + cursor] (coalesced per query).
template <int SHAPE, int MODE>
__device__ __forceinline__ void struct_buffer(StructShared& SS, const float4 P, u32 qmask, int lane, float lo_thr,
                                              float hi_thr, const double* __restrict__ px,
                                              const double* __restrict__ py, const double* __restrict__ pz,
                                              double r, double r2, u32* __restrict__ singles, u64 srow,
                                              u32& ns) {
    constexpr bool FILL = MODE != 0;
    constexpr bool kPacked = SHAPE == LO_SPHERE || SHAPE == LO_CIRCLE;
    PtShared& S = SS.pt;
    const u32 idx = __float_as_uint(P.w);
    const u32 sw = SS.sw[lane];
    const u32 lt = (1u << lane) - 1u;
    const u32 lo_bits = __float_as_uint(lo_thr);
    const u32 band_bits = __float_as_uint(hi_thr) - lo_bits;
    const u64 PX = pack2(P.x, P.x), PY = pack2(P.y, P.y), PZ = pack2(P.z, P.z);
    if (!FILL && kPacked) {
        u32 qm = (qmask | (qmask >> 1) | (qmask >> 2) | (qmask >> 3)) & 0x11111111u;
        S.msk[lane] = 0u;
        __syncwarp();
        while (qm) {
            const int b = __ffs(qm) - 1;
            qm &= qm - 1;
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
            float v[4];
            unpack2(da, v[0], v[1]);
            unpack2(db, v[2], v[3]);
            bool wq[4];
            u32 in[4];
            u32 wband = ~0u;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                wq[t] = (sw >> (b + t)) & 1u;
                in[t] = __ballot_sync(~0u, wq[t] && v[t] < lo_thr);
                if (wq[t]) wband = min(wband, __float_as_uint(v[t]) - lo_bits);
            }
            if (__any_sync(~0u, wband < band_bits)) {  // rare: band points, FP64 decides
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const u32 h = __ballot_sync(~0u, wq[t] && v[t] < hi_thr);
                    if (h ^ in[t]) in[t] = band_fix<SHAPE>(in[t], h ^ in[t], S, b + t, lane, idx, px, py, pz, r, r2);
                }
            }
            if (lane == 0) *reinterpret_cast<uint4*>(&S.msk[b]) = make_uint4(in[0], in[1], in[2], in[3]);
        }
        __syncwarp();
        ns += __popc(S.msk[lane]);
        return;
    }
    if (!FILL) {
        S.msk[lane] = 0u;
        __syncwarp();
    }
    u32 pm = (qmask | (qmask >> 1)) & 0x55555555u;
    while (pm) {
        const int b = __ffs(pm) - 1;
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
            v0 = metric_f<SHAPE>(S.qf[b], P);
            v1 = metric_f<SHAPE>(S.qf[b + 1], P);
        }
        const bool w0 = (sw >> b) & 1u, w1 = (sw >> (b + 1)) & 1u;
        u32 in0 = __ballot_sync(~0u, w0 && v0 < lo_thr);
        u32 in1 = __ballot_sync(~0u, w1 && v1 < lo_thr);
        const u32 h0 = __ballot_sync(~0u, w0 && v0 < hi_thr);
        const u32 h1 = __ballot_sync(~0u, w1 && v1 < hi_thr);
        if (h0 ^ in0) in0 = band_fix<SHAPE>(in0, h0 ^ in0, S, b, lane, idx, px, py, pz, r, r2);
        if (h1 ^ in1) in1 = band_fix<SHAPE>(in1, h1 ^ in1, S, b + 1, lane, idx, px, py, pz, r, r2);
        if (FILL) {
            const u32 c0 = __shfl_sync(~0u, ns, b);
            const u32 c1 = __shfl_sync(~0u, ns, b + 1);
            const u64 s0 = __shfl_sync(~0u, srow, b);
            const u64 s1 = __shfl_sync(~0u, srow, b + 1);
            if ((in0 >> lane) & 1u) singles[s0 + c0 + __popc(in0 & lt)] = idx;
            if ((in1 >> lane) & 1u) singles[s1 + c1 + __popc(in1 & lt)] = idx;
            ns += lane == b ? __popc(in0) : (lane == b + 1 ? __popc(in1) : 0u);
        } else if (lane == 0) {
            *reinterpret_cast<uint2*>(&S.msk[b]) = make_uint2(in0, in1);
        }
    }
    if (!FILL) {
        __syncwarp();
        ns += __popc(S.msk[lane]);
    }
}

#ifndef LO_ST_PREFILTER
#define LO_ST_PREFILTER 1
#endif
// MODE 0: count walk (counts, range / single counts, ranges into per-query scratch slots,
//         per-buffer records for the singles replay);
// MODE 2: full fill walk (ranges + singles) over `tile_list` (overflowed tiles) or every tile.
template <int SHAPE, int MODE>
#ifndef LO_STRUCT_MINB
#define LO_STRUCT_MINB 10
#endif
__global__ void __launch_bounds__(kPtThreads, LO_STRUCT_MINB) struct_pt_kernel(
    const TNodeF* __restrict__ tf, const float4* __restrict__ rbf, const double* __restrict__ rb,
    const float4* __restrict__ pf, const double* __restrict__ px, const double* __restrict__ py,
    const double* __restrict__ pz, Queries q, FloatTest ft, float compact, double r, double r2,
    u32* __restrict__ counts, u32* __restrict__ nrng, u32* __restrict__ nsgl,
    const u64* __restrict__ r_off, u32* __restrict__ ranges, const u64* __restrict__ s_off,
    u32* __restrict__ singles, u64* tile_counter, RecPool rp, const u32* __restrict__ tile_list,
    u64 list_n, u32* __restrict__ rscratch) {
    constexpr bool FILL = MODE != 0;
    __shared__ StructShared shared_s[kPtWarps];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    StructShared& SS = shared_s[w];
    PtShared& S = SS.pt;
    const u64 ntiles = tile_list ? list_n : (q.m + 31) / 32;
    const int cl = lane & 7, grp = lane >> 3;
    constexpr bool kSq = SHAPE == LO_SPHERE || SHAPE == LO_CIRCLE;
    const float lo_thr = kSq ? ft.t_lo : ft.r_lo;
    const float hi_thr = kSq ? ft.t_hi : ft.r_hi;
    u64 chunk_base = 0;  // count pass: this warp's current record chunk (in records)
    u32 chunk_left = 0;
    for (;;) {
        u64 tile = 0;
        if (lane == 0) tile = atomicAdd(reinterpret_cast<unsigned long long*>(tile_counter), 1ull);
        tile = __shfl_sync(~0u, tile, 0);
        if (tile >= ntiles) break;
        if (tile_list) tile = tile_list[tile];
        if (MODE == 0 && rp.pool && chunk_left < rp.cap) {
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
        float4 qf = make_float4(INFINITY, INFINITY, INFINITY, 0.f);
        if (active) {
            load_query(q, qi, cx, cy, cz);
            qf = load_query_f(q, qi);
        }
        __syncwarp();
        S.qf[lane] = qf;
        S.qx[lane] = qf.x;
        S.qy[lane] = qf.y;
        S.qz[lane] = qf.z;
        S.qd[lane][0] = cx;
        S.qd[lane][1] = cy;
        S.qd[lane][2] = cz;
        u32 count = 0, nr = 0, ns = 0, last_e = 0, skip_end = 0;
        u32* rrow = nullptr;
        u64 srow = 0;
        if (FILL && active) {
            rrow = ranges + 2 * r_off[qi];
            srow = s_off[qi];
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
#if LO_ST_PREFILTER
        // the whole tile's query box for the leaf-point prefilter (as in the lin walk)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            float tl = fminf(gl[a], __shfl_xor_sync(~0u, gl[a], 8));
            float th = fmaxf(gh[a], __shfl_xor_sync(~0u, gh[a], 8));
            tl = fminf(tl, __shfl_xor_sync(~0u, tl, 16));
            th = fmaxf(th, __shfl_xor_sync(~0u, th, 16));
            if (lane == 0) S.tbox[a] = tl, S.tbox[3 + a] = th;
        }
#endif
        u32 fill = 0, qmask = 0, nrec = 0;
        u32* rec_tile = (MODE == 0 && rp.pool && chunk_left >= rp.cap) ? rp.pool + chunk_base * 64 : nullptr;
        auto flush = [&]() {
            // the buffer's 32 points are loaded at once (one latency per buffer, not per leaf);
            // slots >= fill get +INF coordinates and an empty want mask
            float4 P = make_float4(INFINITY, INFINITY, INFINITY, 0.f);
            if (static_cast<u32>(lane) < fill) {
                const u32 g = S.bix[lane];
                P = __ldg(pf + g);
                P.w = __uint_as_float(g);
            }
            struct_buffer<SHAPE, MODE>(SS, P, qmask, lane, lo_thr, hi_thr, px, py, pz, r, r2, singles, srow, ns);
            if (MODE == 0 && rec_tile) {
                if (nrec < rp.cap) {
                    u32* R = rec_tile + nrec * 64;
                    R[lane] = __float_as_uint(P.w);
                    R[32 + lane] = S.msk[lane];
                }
                ++nrec;
            }
        };
        int sp = 1;
        if (lane == 0) S.stack[0] = 0;
        __syncwarp();
        while (sp > 0) {
            const u32 t = S.stack[--sp];
            const NodeF nd = load_node_f(tf, t);
            // this lane's relation to the node's reference octant box
            int rel = kDisjoint;
            const bool live = active && nd.begin >= skip_end;
            if (live) {
                const float4 blo = __ldg(rbf + 2 * static_cast<u64>(t));
                const float4 bhi = __ldg(rbf + 2 * static_cast<u64>(t) + 1);
                rel = classify_ref_f<SHAPE>(qf, blo, bhi, ft);
                if (rel == kRelU) {
                    NodeView box;
                    const double* bb = rb + 6 * static_cast<u64>(t);
#pragma unroll
                    for (int a = 0; a < 3; ++a) box.lo[a] = __ldg(bb + a), box.hi[a] = __ldg(bb + 3 + a);
                    rel = relation<SHAPE>(cx, cy, cz, r, r2, box);
                }
                if (rel == kContains) {
                    // count pass: ranges go to this query's scratch slots (copied after the scan)
                    u32* rs_q = MODE == 0 && rscratch ? rscratch + 2 * static_cast<u64>(qi) * kStructRangeCap : nullptr;
                    if (nr > 0 && last_e == nd.begin) {
                        if (FILL) rrow[2 * (nr - 1) + 1] = nd.end;
                        else if (rs_q && nr <= kStructRangeCap) rs_q[2 * (nr - 1) + 1] = nd.end;
                    } else {
                        if (FILL) rrow[2 * nr] = nd.begin, rrow[2 * nr + 1] = nd.end;
                        else if (rs_q && nr < kStructRangeCap) rs_q[2 * nr] = nd.begin, rs_q[2 * nr + 1] = nd.end;
                        ++nr;
                    }
                    last_e = nd.end;
                    count += nd.end - nd.begin;
                }
                if (rel != kIntersects) skip_end = nd.end;  // Contains / Disjoint: not descended
            }
            const u32 inter = __ballot_sync(~0u, rel == kIntersects);
            if (!inter) continue;
            if (nd.nchild != 0) {
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
                u32 sb = __ballot_sync(~0u, keep);
                sb = (sb | (sb >> 8) | (sb >> 16) | (sb >> 24)) & 0xffu;
                const int k = __popc(sb);
                __syncwarp();
                if (lane < 8 && ((sb >> lane) & 1u))
                    S.stack[sp + k - 1 - __popc(sb & ((1u << lane) - 1u))] = nd.child0 + lane;
                sp += k;
                __syncwarp();
                continue;
            }
            // leaf: its points, wanted by the lanes that found it Intersects
#if LO_ST_PREFILTER
            // a point farther than r from the tile's query box is a single of no tile query: dropped
            // before it takes a buffer slot (survivors keep point order, so singles stay ascending)
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
                if (ok && pos < 32) S.bix[pos] = g, SS.sw[pos] = inter;
                fill += __popc(bal);
                qmask |= inter;
                if (fill >= 32) {
                    const u32 over = fill - 32;
                    fill = 32;
                    __syncwarp();
                    flush();
                    __syncwarp();
                    if (ok && pos >= 32) S.bix[pos - 32] = g, SS.sw[pos - 32] = inter;
                    fill = over;
                    qmask = over ? inter : 0u;
                }
            }
#else
            for (u32 base = nd.begin; base < nd.end;) {
                const u32 take = min(32u - fill, nd.end - base);
                __syncwarp();
                if (static_cast<u32>(lane) < take) {
                    S.bix[fill + lane] = base + lane;
                    SS.sw[fill + lane] = inter;
                }
                fill += take;
                qmask |= inter;
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
        if (fill) {
            __syncwarp();
            if (static_cast<u32>(lane) >= fill) SS.sw[lane] = 0;
            __syncwarp();
            flush();
        }
        if (MODE == 0 && active) {
            counts[qi] = count + ns;
            nrng[qi] = nr;
            nsgl[qi] = ns;
        }
        if (MODE == 0 && rp.pool) {
            // a query with more ranges than its scratch slots sends the tile to the fill walk
            const bool rovf = __any_sync(~0u, rscratch && nr > kStructRangeCap);
            const bool ok = rec_tile && nrec <= rp.cap && !rovf;
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

static bool struct_float_path(const lo_octree* t, const lo_coded* c, const Queries& q, double r) {
    return make_float_test(r, std::max(c->bmax, q.bmax)).enabled && q.f && t->tf && c->pf && t->rbf &&
           !force_fp64();
}

// MODE 0 count (+ records, range slots), 2 full fill walk (over `list` when given).
template <int MODE>
static void launch_struct_pt(lo_context* ctx, int shape, const lo_octree* t, const lo_coded* c, const Queries& q,
                             double r, lo_csr* out, u32* nrng, u32* nsgl, RecPool rp = RecPool{},
                             const u32* list = nullptr, u64 list_n = 0, u32* rscratch = nullptr) {
    const double r2 = r * r;  // SearchKernel ctor (geometry.hpp:107)
    const u64 tiles = list ? list_n : (q.m + 31) / 32;
    const FloatTest ft = make_float_test(r, std::max(c->bmax, q.bmax));
    u64* counter = dalloc_t<u64>(ctx, 1);
    LO_CUDA(cudaMemsetAsync(counter, 0, 8, ctx->stream));
    const int pblocks = static_cast<int>(std::max<u64>(
        1, std::min<u64>((tiles + kPtWarps - 1) / kPtWarps, static_cast<u64>(ctx->sm_count) * LO_STRUCT_MINB)));
    static const double compact_mul = [] {  // as in the Lin walk (radius.cu)
        const char* e = std::getenv("LO_COMPACT_MUL");
        return e ? std::strtod(e, nullptr) : 8.0;
    }();
    const float compact = static_cast<float>(compact_mul * r);
#define LO_STRUCT_PT(S)                                                                                 \
    case S:                                                                                             \
        struct_pt_kernel<S, MODE><<<pblocks, kPtThreads, 0, ctx->stream>>>(                             \
            t->tf, t->rbf, t->rb, c->pf, c->x, c->y, c->z, q, ft, compact, r, r2, out->counts, nrng,     \
            nsgl, out->range_offsets, out->ranges, out->single_offsets, out->singles, counter, rp, list, \
            list_n, rscratch);                                                                          \
        break;
    switch (shape) {
        LO_STRUCT_PT(LO_SPHERE)
        LO_STRUCT_PT(LO_CIRCLE)
        LO_STRUCT_PT(LO_CUBE)
        LO_STRUCT_PT(LO_SQUARE)
        default: throw Error(LO_INVALID_ARGUMENT, "unknown kernel shape");
    }
#undef LO_STRUCT_PT
    LO_CHECK_LAUNCH();
    dfree(ctx, counter);
}

// The exact FP64 fallback (the FP32 filter disabled for this radius / cloud extent).
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
    ensure_float_shadows(ctx, c, t);
    ensure_ref_boxes(ctx, c, t);
    auto* out = new lo_csr;
    out->ctx = ctx;
    out->rows = q.m;
    out->is_struct = true;
    u32 *nrng = nullptr, *nsgl = nullptr, *rscratch = nullptr;
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
        const bool fast = q.m && struct_float_path(t, c, q, r);
        RecSetup rs;
        if (fast) {
            try {
                rs = setup_records(ctx, (q.m + 31) / 32, rec_cap());
                rscratch = dalloc_t<u32>(ctx, 2 * q.m * kStructRangeCap);
            } catch (const Error&) {  // no room for records / range slots: fill walks instead
                rs = RecSetup{};
                dfree(ctx, rscratch);
                rscratch = nullptr;
            }
        }
        stage_begin(ctx, "struct_count");
        if (fast)
            launch_struct_pt<0>(ctx, shape, t, c, q, r, out, nrng, nsgl, rs.rp, nullptr, 0, rscratch);
        else if (q.m)
            launch_struct<false>(ctx, shape, t, c, q, r, out, nrng, nsgl);
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
        if (fast && rs.rp.pool) {
            // singles: replay of the count pass's records (want-masked memberships); ranges: a
            // walk without leaf points; overflowed tiles: the full fill walk
            const u32 n_ovf = replay_records(ctx, rs, q.m, out->single_offsets, out->singles, out->total_singles);
            if (out->total_ranges) {
                struct_copy_ranges<<<grid_rows(ctx, q.m * kStructRangeCap), 256, 0, ctx->stream>>>(
                    rscratch, nrng, q.m, out->range_offsets, rs.rp.rec_n, out->ranges);
                LO_CHECK_LAUNCH();
            }
            if (n_ovf) launch_struct_pt<2>(ctx, shape, t, c, q, r, out, nrng, nsgl, RecPool{}, rs.ovf, n_ovf);
        } else if (fast) {
            launch_struct_pt<2>(ctx, shape, t, c, q, r, out, nrng, nsgl);
        } else if (q.m) {
            launch_struct<true>(ctx, shape, t, c, q, r, out, nrng, nsgl);
        }
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
        dfree(ctx, rscratch);
        free_csr_buffers(ctx, out);
        delete out;
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
        throw;
    }
    dfree(ctx, nrng);
    dfree(ctx, nsgl);
    dfree(ctx, rscratch);
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

// Releases a result's buffers in order behind their last reader: a pending async download
// (whose stream waited for the digests), else pending digests on the aux stream, else ctx->stream.
// Buffers from big_alloc are parked in the context cache; the rest are freed (deferred if guarded).
void free_csr_buffers(lo_context* ctx, lo_csr* csr) {
    auto pending = [](cudaEvent_t& e) {
        if (!e) return false;
        const bool busy = cudaEventQuery(e) != cudaSuccess;
        if (busy) cudaGetLastError();  // cudaErrorNotReady is not an error
        cudaEventDestroy(e);  // released once recorded work completes
        e = nullptr;
        return busy;
    };
    cudaStream_t last = ctx->stream;
    unsigned guarded = 0;
    const bool aux_digests = csr->digested != nullptr;
    if (pending(csr->copied)) {
        last = ctx->copy_stream;
        // the copied buffers, and with aux-stream digests also what the digests read (the copy
        // stream waited for them); inline digests finished on ctx->stream already
        guarded = csr->copy_mask | (aux_digests ? 2u | 4u | 8u : 0u);
    }
    if (pending(csr->digested) && !guarded) {
        last = ctx->aux_stream;
        guarded = 2u | 4u | 8u;  // fps, offsets, indices
    }
    csr->copy_mask = 0;
    void** bufs[4] = {reinterpret_cast<void**>(&csr->counts), reinterpret_cast<void**>(&csr->fps),
                      reinterpret_cast<void**>(&csr->offsets), reinterpret_cast<void**>(&csr->indices)};
    for (int b = 0; b < 4; ++b) {
        if (!*bufs[b]) continue;
        const cudaStream_t s = (guarded >> b) & 1u ? last : ctx->stream;
        if (csr->cap[b])
            big_release(ctx, *bufs[b], csr->cap[b], s);
        else if (s == ctx->stream)
            dfree(ctx, *bufs[b]);
        else
            big_release(ctx, *bufs[b], 0, s);  // deferred behind the reader
        *bufs[b] = nullptr;
        csr->cap[b] = 0;
    }
    dfree(ctx, csr->range_offsets);
    dfree(ctx, csr->ranges);
    dfree(ctx, csr->single_offsets);
    dfree(ctx, csr->singles);
    csr->range_offsets = nullptr, csr->ranges = nullptr, csr->single_offsets = nullptr;
    csr->singles = nullptr;
}

}  // namespace lo
