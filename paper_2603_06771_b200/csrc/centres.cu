// centres.cu -- explicit centre lists (BatchMode::RandomSubset, search.cpp:273-283; any caller
// order, e.g. the cfg4 "original order") are searched in SFC order and the rows put back.
//
// The search kernels give one warp 32 consecutive queries and walk the union of their
// traversals; that is cheap when the 32 queries are spatial neighbours (Full mode) and ruinous
// when they are scattered (cfg4 original order: radius 15x, kNN 600x slower).  Centres are cloud
// indices of the SFC-sorted cloud, so sorting them by value IS sorting them along the curve:
// one stable radix sort (payload = position), search, then scatter rows / counts / digests back
// to the caller's order.
#include <cstring>
#include <algorithm>
#include <vector>

#include "lo_internal.cuh"

namespace lo {

__global__ void widen_u32(const u32* __restrict__ in, u64 n, u64* __restrict__ out) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        out[i] = in[i];
}

__global__ void narrow_u64(const u64* __restrict__ in, u64 n, u32* __restrict__ out) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        out[i] = static_cast<u32>(in[i]);
}

// byte-digit histograms of u32 keys (digits 0..3; digit 4 of the widened key is all zero)
__global__ void digit_hist_u32(const u32* __restrict__ keys, u64 n, u32* __restrict__ hist) {
    __shared__ u32 h[4 * 256];
    for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) h[i] = 0;
    __syncthreads();
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u32 k = keys[i];
#pragma unroll
        for (int d = 0; d < 4; ++d) atomicAdd(&h[d * 256 + ((k >> (8 * d)) & 0xffu)], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x)
        if (h[i]) atomicAdd(&hist[i], h[i]);
}

static int grid_n(lo_context* ctx, u64 n) {
    return static_cast<int>(std::max<u64>(1, std::min<u64>((n + 255) / 256, ctx->sm_count * 16ull)));
}

SortedCentres sort_centres(lo_context* ctx, const u32* centres, u64 m) {
    SortedCentres s;
    if (m == 0) return s;
    stage_begin(ctx, "centre_sort");
    u64* k64 = dalloc_t<u64>(ctx, m);
    u64* ks = nullptr;
    u32* hist = nullptr;
    try {
        s.idx = dalloc_t<u32>(ctx, m);
        s.pos = dalloc_t<u32>(ctx, m);
        ks = dalloc_t<u64>(ctx, m);
        hist = dalloc_t<u32>(ctx, 4 * 256);
        LO_CUDA(cudaMemsetAsync(hist, 0, 4 * 256 * 4, ctx->stream));
        widen_u32<<<grid_n(ctx, m), 256, 0, ctx->stream>>>(centres, m, k64);
        LO_CHECK_LAUNCH();
        digit_hist_u32<<<std::min(grid_n(ctx, m), ctx->sm_count * 2), 256, 0, ctx->stream>>>(centres, m, hist);
        LO_CHECK_LAUNCH();
        std::vector<u32> hh(8 * 256, 0);
        fetch_small(ctx, hist, 4 * 256 * 4);
        std::memcpy(hh.data(), ctx->pinned_scratch, 4 * 256 * 4);
        hh[4 * 256] = static_cast<u32>(m);  // digit 4 (bits 32..39) is constant
        radix_sort(ctx, k64, m, hh.data(), 11, ks, s.pos);  // 11 levels = 33 bits -> 5 passes
        narrow_u64<<<grid_n(ctx, m), 256, 0, ctx->stream>>>(ks, m, s.idx);
        LO_CHECK_LAUNCH();
    } catch (...) {
        dfree(ctx, k64), dfree(ctx, ks), dfree(ctx, hist);
        dfree(ctx, s.idx), dfree(ctx, s.pos);
        throw;
    }
    dfree(ctx, k64), dfree(ctx, ks), dfree(ctx, hist);
    stage_end(ctx);
    return s;
}

// ---- kNN rows: fixed width, scatter row i to row pos[i] --------------------------------------
__global__ void scatter_knn_rows(const u32* __restrict__ pos, u64 m, u32 k, const u32* __restrict__ idx_s,
                                 const double* __restrict__ dist_s, const u64* __restrict__ fps_s,
                                 u32* __restrict__ idx_o, double* __restrict__ dist_o, u64* __restrict__ fps_o) {
    const u64 total = m * k;
    for (u64 e = blockIdx.x * (u64)blockDim.x + threadIdx.x; e < total; e += (u64)gridDim.x * blockDim.x) {
        const u64 i = e / k, j = e - i * k;
        const u64 o = static_cast<u64>(pos[i]) * k + j;
        idx_o[o] = idx_s[e];
        dist_o[o] = dist_s[e];
        if (fps_s && j == 0) fps_o[pos[i]] = fps_s[i];
    }
}

void unsort_knn(lo_context* ctx, const SortedCentres& s, lo_knn_result* r) {
    const u64 m = r->rows, k = r->keff;
    if (m == 0) return;
    stage_begin(ctx, "centre_unsort");
    u32* idx = dalloc_t<u32>(ctx, m * k);
    double* dist = nullptr;
    u64* fps = nullptr;
    try {
        dist = dalloc_t<double>(ctx, m * k);
        if (r->fps) fps = dalloc_t<u64>(ctx, m);
        scatter_knn_rows<<<grid_n(ctx, m * k), 256, 0, ctx->stream>>>(s.pos, m, static_cast<u32>(k), r->idx,
                                                                       r->dist, r->fps, idx, dist, fps);
        LO_CHECK_LAUNCH();
    } catch (...) {
        dfree(ctx, idx), dfree(ctx, dist), dfree(ctx, fps);
        throw;
    }
    dfree(ctx, r->idx), dfree(ctx, r->dist), dfree(ctx, r->fps);
    r->idx = idx, r->dist = dist, r->fps = fps;
    stage_end(ctx);
}

// ---- CSR rows: counts / digests scattered, offsets rescanned, rows copied by warps ---------
__global__ void scatter_u32(const u32* __restrict__ pos, u64 m, const u32* __restrict__ in, u32* __restrict__ out) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < m; i += (u64)gridDim.x * blockDim.x)
        out[pos[i]] = in[i];
}
__global__ void scatter_u64(const u32* __restrict__ pos, u64 m, const u64* __restrict__ in, u64* __restrict__ out) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < m; i += (u64)gridDim.x * blockDim.x)
        out[pos[i]] = in[i];
}
__global__ void row_lengths(const u64* __restrict__ off, u64 m, u32* __restrict__ len) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < m; i += (u64)gridDim.x * blockDim.x)
        len[i] = static_cast<u32>(off[i + 1] - off[i]);
}
// row i of (off_s, data_s) -> row pos[i] of (off_o, data_o); `w` u32 words per element
__global__ void copy_rows(const u32* __restrict__ pos, u64 m, const u64* __restrict__ off_s,
                          const u32* __restrict__ data_s, const u64* __restrict__ off_o,
                          u32* __restrict__ data_o, u32 w) {
    const int lane = threadIdx.x & 31;
    for (u64 i = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; i < m;
         i += ((u64)gridDim.x * blockDim.x) >> 5) {
        const u64 b = off_s[i] * w, e = off_s[i + 1] * w;
        const u64 o = off_o[pos[i]] * w;
        for (u64 j = b + lane; j < e; j += 32) data_o[o + (j - b)] = data_s[j];
    }
}

// Re-orders one CSR (off[m+1], data) whose rows follow the sorted centres; returns the new pair.
static void unsort_csr_part(lo_context* ctx, const SortedCentres& s, u64 m, u64*& off, u32*& data, u64 total,
                            u32 w) {
    u32* len_s = dalloc_t<u32>(ctx, m);
    u32* len_o = nullptr;
    u64* off_o = nullptr;
    u32* data_o = nullptr;
    try {
        len_o = dalloc_t<u32>(ctx, m);
        off_o = dalloc_t<u64>(ctx, m + 1);
        data_o = dalloc_t<u32>(ctx, total * w);
        row_lengths<<<grid_n(ctx, m), 256, 0, ctx->stream>>>(off, m, len_s);
        LO_CHECK_LAUNCH();
        scatter_u32<<<grid_n(ctx, m), 256, 0, ctx->stream>>>(s.pos, m, len_s, len_o);
        LO_CHECK_LAUNCH();
        exclusive_scan_u32_to_u64(ctx, len_o, off_o, m);
        if (total) {
            copy_rows<<<static_cast<int>(std::min<u64>((m * 32 + 255) / 256, ctx->sm_count * 16ull)), 256, 0,
                        ctx->stream>>>(s.pos, m, off, data, off_o, data_o, w);
            LO_CHECK_LAUNCH();
        }
    } catch (...) {
        dfree(ctx, len_s), dfree(ctx, len_o), dfree(ctx, off_o), dfree(ctx, data_o);
        throw;
    }
    dfree(ctx, len_s), dfree(ctx, len_o);
    dfree(ctx, off), dfree(ctx, data);
    off = off_o, data = data_o;
}

void unsort_csr(lo_context* ctx, const SortedCentres& s, lo_csr* c) {
    const u64 m = c->rows;
    if (c->digested) {  // the row digests are still being computed on the aux stream
        LO_CUDA(cudaStreamWaitEvent(ctx->stream, c->digested, 0));
        cudaEventDestroy(c->digested);
        c->digested = nullptr;
    }
    if (m == 0) return;
    stage_begin(ctx, "centre_unsort");
    u32* counts = dalloc_t<u32>(ctx, m);
    scatter_u32<<<grid_n(ctx, m), 256, 0, ctx->stream>>>(s.pos, m, c->counts, counts);
    LO_CHECK_LAUNCH();
    dfree(ctx, c->counts);
    c->counts = counts;
    if (c->fps) {
        u64* fps = dalloc_t<u64>(ctx, m);
        scatter_u64<<<grid_n(ctx, m), 256, 0, ctx->stream>>>(s.pos, m, c->fps, fps);
        LO_CHECK_LAUNCH();
        dfree(ctx, c->fps);
        c->fps = fps;
    }
    if (c->is_struct) {
        unsort_csr_part(ctx, s, m, c->range_offsets, c->ranges, c->total_ranges, 2);
        unsort_csr_part(ctx, s, m, c->single_offsets, c->singles, c->total_singles, 1);
        // the expanded CSR is rebuilt on demand from the re-ordered parts
        dfree(ctx, c->indices);
        c->indices = nullptr;
        exclusive_scan_u32_to_u64(ctx, c->counts, c->offsets, m);
    } else {
        unsort_csr_part(ctx, s, m, c->offsets, c->indices, c->total, 1);
    }
    for (auto& b : c->cap) b = 0;  // replaced (or stream-ordered) buffers: plain frees from here on
    stage_end(ctx);
    sync(ctx);
}

__global__ void gather_q(const u32* __restrict__ pos, u64 m, const double* __restrict__ x,
                         const double* __restrict__ y, const double* __restrict__ z, const float4* __restrict__ f,
                         double* __restrict__ x2, double* __restrict__ y2, double* __restrict__ z2,
                         float4* __restrict__ f2) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < m; i += (u64)gridDim.x * blockDim.x) {
        const u32 j = pos[i];
        x2[i] = x[j], y2[i] = y[j], z2[i] = z[j], f2[i] = f[j];
    }
}

void gather_queries(lo_context* ctx, const u32* pos, u64 m, double*& x, double*& y, double*& z, float4*& f) {
    if (m == 0) return;
    double* x2 = dalloc_t<double>(ctx, m);
    double* y2 = dalloc_t<double>(ctx, m);
    double* z2 = dalloc_t<double>(ctx, m);
    float4* f2 = dalloc_t<float4>(ctx, m);
    gather_q<<<grid_n(ctx, m), 256, 0, ctx->stream>>>(pos, m, x, y, z, f, x2, y2, z2, f2);
    LO_CHECK_LAUNCH();
    dfree(ctx, x), dfree(ctx, y), dfree(ctx, z), dfree(ctx, f);
    x = x2, y = y2, z = z2, f = f2;
}

}  // namespace lo
