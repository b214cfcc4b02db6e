// context.cu -- contexts, errors, device memory, stage timers, exclusive scans, host tables.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include <algorithm>
#include <chrono>
#include <atomic>
#include <cstdio>
#include <mutex>

#include "lo_internal.cuh"

namespace lo {

thread_local std::string g_last_error;
void set_last_error(const char* m) { g_last_error = m; }

static std::atomic<unsigned long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
    char buf[512];
    std::snprintf(buf, sizeof buf, "CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e),
                  cudaGetErrorString(e), what, file, line);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();  // clear the sticky-free allocation error
        throw Error(LO_OUT_OF_MEMORY, buf);
    }
    throw Error(LO_CUDA_ERROR, buf);
}

void reclaim(lo_context* ctx, bool wait) {
    SlowLog slow("reclaim", ctx->deferred.size());
    auto& d = ctx->deferred;
    for (size_t i = 0; i < d.size();) {
        if (wait) cudaEventSynchronize(d[i].done);
        if (cudaEventQuery(d[i].done) == cudaSuccess) {
            for (void* p : d[i].ptrs) cudaFreeAsync(p, ctx->stream);
            cudaEventDestroy(d[i].done);
            d[i] = d.back();
            d.pop_back();
        } else {
            cudaGetLastError();  // cudaErrorNotReady is not an error
            ++i;
        }
    }
}

// Large device buffers (>= 64 MB) are recycled by the context instead of the stream-ordered pool.
// A step of the hot path allocates and frees the same ~25 large buffers every time (the coded cloud's
// SoA arrays, the sort's ping-pong arrays, the tree's tables, the 25 GB CSR...), and whenever the pool
// has no free block of the right shape it maps new physical memory inside cudaMallocAsync: 2-4 ms
// per 400-800 MB and 140 ms for the 25 GB CSR, with the GPU idle meanwhile -- cfg3 steps varied
// between 85 and 117 ms on identical kernels.  dalloc() hands out a parked buffer of the right size
// when there is one; dfree() / big_release() park it again (behind an event when its last reader is
// another stream).  Parked buffers go back to the pool when the cache is over its limit, on
// lo_context_synchronize, or when an allocation fails.
constexpr size_t kBigBytes = 64ull << 20;
constexpr size_t kCacheEntries = 48;
// parked bytes are capped too (oldest finished first): what the cache holds the pool cannot reuse
// for other shapes, and a pool that has to grow is what made the allocations slow
static size_t cache_byte_cap(lo_context* ctx) {
    if (!ctx->cache_cap) {
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
            cudaGetLastError();
            total_b = 64ull << 30;
        }
        ctx->cache_cap = total_b / 2;
    }
    return ctx->cache_cap;
}

static bool cache_ready(const lo_context::Cached& c) {
    if (!c.ready) return true;  // last used on ctx->stream: stream order makes it reusable
    if (cudaEventQuery(c.ready) == cudaSuccess) return true;
    cudaGetLastError();  // cudaErrorNotReady is not an error
    return false;
}

static void cache_free(lo_context* ctx, lo_context::Cached& c) {
    if (c.ready) {
        cudaEventSynchronize(c.ready);
        cudaEventDestroy(c.ready);
    }
    cudaFreeAsync(c.p, ctx->stream);
}

void cache_drain(lo_context* ctx) {
    for (auto& c : ctx->cache) cache_free(ctx, c);
    ctx->cache.clear();
}

static void* pool_alloc(lo_context* ctx, size_t bytes) {
    void* p = nullptr;
    static const bool dbg_alloc = std::getenv("LO_DEBUG_ALLOC") != nullptr;
    const auto t0 = dbg_alloc ? std::chrono::steady_clock::now() : std::chrono::steady_clock::time_point{};
    cudaError_t e = cudaMallocAsync(&p, bytes, ctx->stream);
    if (e != cudaSuccess && !ctx->cache.empty()) {  // parked buffers go back first
        cudaGetLastError();
        if (dbg_alloc) std::fprintf(stderr, "[lo] alloc %zu B failed: draining %zu parked buffers\n", bytes, ctx->cache.size());
        cache_drain(ctx);
        e = cudaMallocAsync(&p, bytes, ctx->stream);
    }
    if (dbg_alloc) {
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (ms > 0.2) std::fprintf(stderr, "[lo] cudaMallocAsync %zu B took %.2f ms\n", bytes, ms);
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        char buf[160];
        std::snprintf(buf, sizeof buf, "device allocation of %zu bytes failed (%s)", bytes, cudaGetErrorName(e));
        throw Error(LO_OUT_OF_MEMORY, buf);
    }
    return p;
}

void* dalloc(lo_context* ctx, size_t bytes) {
    SlowLog slow("dalloc", bytes);
    if (!ctx->deferred.empty()) reclaim(ctx, false);
    if (bytes < kBigBytes) return pool_alloc(ctx, bytes);
    auto& c = ctx->cache;
    int best = -1;
    for (size_t i = 0; i < c.size(); ++i) {
        if (c[i].bytes < bytes || c[i].bytes > bytes + bytes / 2 + kBigBytes) continue;
        if (!cache_ready(c[i])) continue;
        if (best < 0 || c[i].bytes < c[best].bytes) best = static_cast<int>(i);
    }
    void* p;
    size_t got = bytes;
    if (best >= 0) {
        p = c[best].p;
        got = c[best].bytes;
        if (c[best].ready) cudaEventDestroy(c[best].ready);
        c.erase(c.begin() + best);
    } else {
        p = pool_alloc(ctx, bytes);
    }
    ctx->big[p] = got;
    return p;
}

void* big_alloc(lo_context* ctx, size_t bytes, size_t* got) {
    void* p = dalloc(ctx, bytes);
    const auto it = ctx->big.find(p);
    *got = it != ctx->big.end() ? it->second : 0;  // 0: a small buffer (plain pool)
    return p;
}

// Parks a large buffer (its last reader: `last_use`), trimming the cache to its limit.
static void park(lo_context* ctx, void* p, size_t bytes, cudaStream_t last_use) {
    SlowLog slow("park", bytes);
    lo_context::Cached c{p, bytes, nullptr};
    if (last_use != ctx->stream) {
        LO_CUDA(cudaEventCreateWithFlags(&c.ready, cudaEventDisableTiming));
        LO_CUDA(cudaEventRecord(c.ready, last_use));
    }
    auto& cache = ctx->cache;
    cache.push_back(c);
    size_t parked = 0;
    for (const auto& e : cache) parked += e.bytes;
    const size_t cap = cache_byte_cap(ctx);
    // over the limits the oldest finished buffers go back to the pool (waiting only if none has)
    for (size_t i = 0; i < cache.size() && (cache.size() > kCacheEntries || parked > cap);) {
        if (cache_ready(cache[i])) {
            parked -= cache[i].bytes;
            cache_free(ctx, cache[i]);
            cache.erase(cache.begin() + i);
        } else {
            ++i;
        }
    }
    while (cache.size() > 2 * kCacheEntries) {
        cache_free(ctx, cache.front());
        cache.erase(cache.begin());
    }
}

void big_release(lo_context* ctx, void* p, size_t /*bytes*/, cudaStream_t last_use) {
    if (!p) return;
    const auto it = ctx->big.find(p);
    if (it != ctx->big.end()) {
        const size_t size = it->second;
        ctx->big.erase(it);
        park(ctx, p, size, last_use);
        return;
    }
    if (last_use == ctx->stream) {
        cudaFreeAsync(p, ctx->stream);
    } else {  // release once the other stream's reader has finished
        lo_context::Deferred d{nullptr, {p}};
        LO_CUDA(cudaEventCreateWithFlags(&d.done, cudaEventDisableTiming));
        LO_CUDA(cudaEventRecord(d.done, last_use));
        ctx->deferred.push_back(std::move(d));
    }
}

void dfree(lo_context* ctx, void* p) {
    if (!p) return;
    const auto it = ctx->big.find(p);
    if (it != ctx->big.end()) {
        const size_t size = it->second;
        ctx->big.erase(it);
        park(ctx, p, size, ctx->stream);
        return;
    }
    cudaFreeAsync(p, ctx->stream);
}

// Host waits inside a batch (a histogram or total the host needs next) spin on an event query
// instead of cudaStreamSynchronize: a blocking wait may sleep the thread, and its wake-up latency
// left the GPU idle at each of the ~8 such points of a step -- identical kernels, cfg3 steps of 85
// or 91-93 ms depending on the run.
void spin_wait(cudaEvent_t ev) {
    for (;;) {
        const cudaError_t e = cudaEventQuery(ev);
        if (e == cudaSuccess) return;
        if (e != cudaErrorNotReady) LO_CUDA(e);
    }
}

void sync(lo_context* ctx) {
    if (!ctx->sync_ev) LO_CUDA(cudaEventCreateWithFlags(&ctx->sync_ev, cudaEventDisableTiming));
    LO_CUDA(cudaEventRecord(ctx->sync_ev, ctx->stream));
    spin_wait(ctx->sync_ev);
}

__global__ void fetch_words(const u32* __restrict__ src, u32* dst, u32 words) {
    for (u32 i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
}

void fetch_small(lo_context* ctx, const void* dev, size_t bytes) {
    require(bytes <= 16384 && bytes % 4 == 0, LO_INVALID_ARGUMENT, "fetch_small size");
    fetch_words<<<1, 256, 0, ctx->stream>>>(static_cast<const u32*>(dev), static_cast<u32*>(ctx->pinned_scratch_dev),
                                          static_cast<u32>(bytes / 4));
    LO_CHECK_LAUNCH();
    sync(ctx);
}

void* arena(lo_context* ctx, size_t bytes) {
    SlowLog slow("arena", bytes);
    if (ctx->arena_bytes >= bytes) return ctx->arena;
    if (ctx->arena) {
        sync(ctx);
        cudaFree(ctx->arena);
        ctx->arena = nullptr;
        ctx->arena_bytes = 0;
    }
    const size_t want = bytes + bytes / 4;  // headroom: a slightly larger batch reuses it
    static const bool debug = std::getenv("LO_DEBUG") != nullptr;
    if (debug) std::fprintf(stderr, "[lo] arena grows to %zu bytes\n", want);
    cudaError_t e = cudaMalloc(&ctx->arena, want);
    if (e != cudaSuccess) {
        cudaGetLastError();
        ctx->arena = nullptr;
        throw Error(LO_OUT_OF_MEMORY, "scratch arena allocation failed");
    }
    ctx->arena_bytes = want;
    return ctx->arena;
}

void stage_begin(lo_context* ctx, const char* name) {
    if (!ctx->timing) return;
    lo_context::Stage s{name, nullptr, nullptr};
    LO_CUDA(cudaEventCreate(&s.a));
    LO_CUDA(cudaEventCreate(&s.b));
    LO_CUDA(cudaEventRecord(s.a, ctx->stream));
    ctx->stages.push_back(s);
}

void stage_end(lo_context* ctx) {
    if (!ctx->timing || ctx->stages.empty()) return;
    LO_CUDA(cudaEventRecord(ctx->stages.back().b, ctx->stream));
}

static void resolve_stages(lo_context* ctx) {
    if (ctx->stages.empty()) return;
    sync(ctx);
    for (auto& s : ctx->stages) {
        float ms = 0.f;
        cudaEventSynchronize(s.b);  // stages may be timed on another stream (broadcast)
        cudaEventElapsedTime(&ms, s.a, s.b);
        ctx->stage_ms.emplace_back(s.name, ms);
        cudaEventDestroy(s.a);
        cudaEventDestroy(s.b);
    }
    ctx->stages.clear();
}

// ---- exclusive scan (3 phases: tile sums, scan of sums, tile scans) ----------------------
constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;

template <class In>
__global__ void __launch_bounds__(kScanThreads) scan_tile_sums(const In* in, u64 n, u64* sums) {
    using BlockReduce = cub::BlockReduce<u64, kScanThreads>;
    __shared__ typename BlockReduce::TempStorage tmp;
    const u64 base = static_cast<u64>(blockIdx.x) * kScanTile;
    u64 acc = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        const u64 j = base + static_cast<u64>(i) * kScanThreads + threadIdx.x;
        if (j < n) acc += in[j];
    }
    const u64 s = BlockReduce(tmp).Sum(acc);
    if (threadIdx.x == 0) sums[blockIdx.x] = s;
}

constexpr int kSumsThreads = 256;
__global__ void __launch_bounds__(kSumsThreads) scan_sums(u64* sums, int nb, u64* total_out) {
    using BlockScan = cub::BlockScan<u64, kSumsThreads>;
    __shared__ typename BlockScan::TempStorage tmp;
    __shared__ u64 carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < nb; base += kSumsThreads) {
        const int j = base + threadIdx.x;
        const u64 v = j < nb ? sums[j] : 0;
        u64 ex, agg;
        BlockScan(tmp).ExclusiveSum(v, ex, agg);
        if (j < nb) sums[j] = ex + carry;
        __syncthreads();
        if (threadIdx.x == 0) carry += agg;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total_out = carry;
}

template <class In, class Out>
__global__ void __launch_bounds__(kScanThreads) scan_tiles(const In* in, u64 n, const u64* sums,
                                                           Out* out) {
    using BlockScan = cub::BlockScan<u64, kScanThreads>;
    __shared__ typename BlockScan::TempStorage tmp;
    __shared__ __align__(16) unsigned char raw[kScanTile * sizeof(Out) > kScanTile * sizeof(In)
                                                   ? kScanTile * sizeof(Out)
                                                   : kScanTile * sizeof(In)];
    In* tile = reinterpret_cast<In*>(raw);
    Out* otile = reinterpret_cast<Out*>(raw);
    const u64 base = static_cast<u64>(blockIdx.x) * kScanTile;
    // coalesced load into shared memory, then each thread scans a blocked run
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        const int t = i * kScanThreads + threadIdx.x;
        const u64 j = base + t;
        tile[t] = j < n ? in[j] : In(0);
    }
    __syncthreads();
    u64 run = 0;
    In v[kScanItems];
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        v[i] = tile[threadIdx.x * kScanItems + i];
        run += v[i];
    }
    u64 ex;
    BlockScan(tmp).ExclusiveSum(run, ex);
    ex += sums[blockIdx.x];
    __syncthreads();
    // write back through shared memory in the output type for coalesced stores
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        otile[threadIdx.x * kScanItems + i] = static_cast<Out>(ex);
        ex += v[i];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        const int t = i * kScanThreads + threadIdx.x;
        const u64 j = base + t;
        if (j < n) out[j] = otile[t];
    }
}

template <class Out>
__global__ void store_total(const u64* s, Out* o) { *o = static_cast<Out>(*s); }

template <class In, class Out>
static void exclusive_scan(lo_context* ctx, const In* in, Out* out, u64 n) {
    const int nb = std::max(1, ceil_div(n, kScanTile));
    u64* sums = dalloc_t<u64>(ctx, nb + 1);
    if (n > 0) {
        scan_tile_sums<In><<<nb, kScanThreads, 0, ctx->stream>>>(in, n, sums);
        LO_CHECK_LAUNCH();
    } else {
        LO_CUDA(cudaMemsetAsync(sums, 0, sizeof(u64), ctx->stream));
    }
    scan_sums<<<1, kSumsThreads, 0, ctx->stream>>>(sums, n > 0 ? nb : 1, sums + nb);
    LO_CHECK_LAUNCH();
    if (n > 0) {
        scan_tiles<In, Out><<<nb, kScanThreads, 0, ctx->stream>>>(in, n, sums, out);
        LO_CHECK_LAUNCH();
    }
    // out[n] = total
    store_total<Out><<<1, 1, 0, ctx->stream>>>(sums + nb, out + n);
    LO_CHECK_LAUNCH();
    dfree(ctx, sums);
}

void exclusive_scan_u32_to_u64(lo_context* ctx, const u32* in, u64* out, u64 n) {
    exclusive_scan<u32, u64>(ctx, in, out, n);
}
void exclusive_scan_u32(lo_context* ctx, const u32* in, u32* out, u64 n) {
    exclusive_scan<u32, u32>(ctx, in, out, n);
}

// ---- curve tables ------------------------------------------------------------------------
// Host Skilling decode (the transpose-to-axes half of the published Hilbert construction the
// reference uses, sfc.cpp:44-73); only used here to derive the descent tables.
static void hilbert_decode_host(u64 code, int level, u32 out[3]) {
    if (level == 0) {
        out[0] = out[1] = out[2] = 0;
        return;
    }
    const u32 mask = (1u << level) - 1;
    u32 a[3] = {compact3(code >> 2) & mask, compact3(code >> 1) & mask, compact3(code) & mask};
    const u32 t = a[2] >> 1;
    a[2] ^= a[1];
    a[1] ^= a[0];
    a[0] ^= t;
    for (u32 q = 2; q != (2u << (level - 1)); q <<= 1) {
        const u32 low = q - 1;
        for (int i = 2; i >= 0; --i) {
            if (a[i] & q) {
                a[0] ^= low;
            } else {
                const u32 s = (a[0] ^ a[i]) & low;
                a[0] ^= s;
                a[i] ^= s;
            }
        }
    }
    out[0] = a[0], out[1] = a[1], out[2] = a[2];
}

static void decode_host(int curve, u64 code, int level, u32 out[3]) {
    if (curve == LO_MORTON) {
        out[0] = compact3(code >> 2), out[1] = compact3(code >> 1), out[2] = compact3(code);
    } else {
        hilbert_decode_host(code, level, out);
    }
}

// Closure of child-digit signatures reachable from the root (same construction as
// CurveStepper, sfc.cpp:157-194), verified by re-decoding every level-5 code.
static CurveTables derive_tables(int curve) {
    CurveTables t{};
    std::vector<u32> sig;
    std::vector<std::pair<u64, int>> ex;
    auto signature = [&](u64 prefix, int depth) {
        u32 s = 0;
        for (int c = 0; c < 8; ++c) {
            u32 cell[3];
            decode_host(curve, prefix * 8 + c, depth + 1, cell);
            s |= (((cell[0] & 1u) << 2) | ((cell[1] & 1u) << 1) | (cell[2] & 1u)) << (3 * c);
        }
        return s;
    };
    auto state_of = [&](u64 prefix, int depth) {
        const u32 s = signature(prefix, depth);
        for (size_t i = 0; i < sig.size(); ++i)
            if (sig[i] == s) return static_cast<int>(i);
        sig.push_back(s);
        ex.emplace_back(prefix, depth);
        require(sig.size() <= 32, LO_LOGIC_ERROR, "curve tables: state set does not close");
        return static_cast<int>(sig.size() - 1);
    };
    state_of(0, 0);
    for (size_t s = 0; s < sig.size(); ++s) {
        for (int c = 0; c < 8; ++c) {
            const int g = (sig[s] >> (3 * c)) & 7;
            const int nx = state_of(ex[s].first * 8 + c, ex[s].second + 1);
            t.dec[s * 8 + c] = static_cast<u8>(g | (nx << 3));
            t.enc[s * 8 + g] = static_cast<u8>(c | (nx << 3));
        }
    }
    t.states = static_cast<int>(sig.size());
    for (int level = 1; level <= 5; ++level) {
        for (u64 code = 0; code < (1ull << (3 * level)); ++code) {
            int s = 0;
            u32 w[3] = {0, 0, 0};
            for (int d = level - 1; d >= 0; --d) {
                const u8 e = t.dec[s * 8 + ((code >> (3 * d)) & 7)];
                w[0] = w[0] << 1 | ((e >> 2) & 1);
                w[1] = w[1] << 1 | ((e >> 1) & 1);
                w[2] = w[2] << 1 | (e & 1);
                s = e >> 3;
            }
            u32 ref[3];
            decode_host(curve, code, level, ref);
            require(w[0] == ref[0] && w[1] == ref[1] && w[2] == ref[2], LO_LOGIC_ERROR,
                    "curve tables disagree with the decoder");
        }
    }
    return t;
}

const CurveTables& curve_tables(int curve) {
    static std::once_flag once;
    static CurveTables tables[2];
    std::call_once(once, [] {
        tables[0] = derive_tables(LO_MORTON);
        tables[1] = derive_tables(LO_HILBERT);
    });
    return tables[curve == LO_MORTON ? 0 : 1];
}

}  // namespace lo

using namespace lo;

// ---- C ABI: context -----------------------------------------------------------------------
extern "C" {

const char* lo_last_error(void) { return g_last_error.c_str(); }
uint64_t lo_launch_count(void) { return g_launches.load(); }
int lo_abi_version(void) { return LO_ABI_VERSION; }

int lo_device_count(int* count) {
    return api([&] {
        int c = 0;
        cudaError_t e = cudaGetDeviceCount(&c);
        if (e != cudaSuccess) {
            cudaGetLastError();
            c = 0;
        }
        *count = c;
    });
}

int lo_context_create(int device, void* stream, lo_context** out) {
    return api([&] {
        int count = 0;
        cudaError_t e = cudaGetDeviceCount(&count);
        if (e != cudaSuccess || count == 0) {
            cudaGetLastError();
            throw Error(LO_NO_DEVICE, "no CUDA device available: the B200 path has no CPU "
                                      "fallback");
        }
        require(device >= 0 && device < count, LO_INVALID_ARGUMENT, "device index out of range");
        LO_CUDA(cudaSetDevice(device));
        cudaDeviceProp prop{};
        LO_CUDA(cudaGetDeviceProperties(&prop, device));
        require(prop.major >= 10, LO_NO_DEVICE,
                "device is not sm_100 class (this library is built for sm_100a only)");
        auto* ctx = new lo_context;
        ctx->device = device;
        ctx->sm_count = prop.multiProcessorCount;
        if (stream) {
            ctx->stream = static_cast<cudaStream_t>(stream);
        } else {
            LO_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
            ctx->own_stream = true;
        }
        LO_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
        LO_CUDA(cudaStreamCreateWithFlags(&ctx->h2d_stream, cudaStreamNonBlocking));
        LO_CUDA(cudaStreamCreateWithFlags(&ctx->aux_stream, cudaStreamNonBlocking));
        for (auto& e : ctx->h2d_done) LO_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        for (auto& e : ctx->d2h_done) LO_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        cudaMemPool_t pool;
        LO_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
        u64 threshold = ~0ull;
        LO_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
        LO_CUDA(cudaHostAlloc(&ctx->pinned_scratch, 16384, cudaHostAllocMapped));
        LO_CUDA(cudaHostGetDevicePointer(&ctx->pinned_scratch_dev, ctx->pinned_scratch, 0));
        curve_tables(LO_HILBERT);  // derive + self-check once
        *out = ctx;
    });
}

int lo_context_destroy(lo_context* ctx) {
    return api([&] {
        if (!ctx) return;
        const int live = ctx->live_handles.load();
        if (live > 0)
            throw Error(LO_LOGIC_ERROR, "lo_context_destroy: " + std::to_string(live) +
                                            " handle(s) created on this context are still alive");
        DeviceGuard dev(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        if (ctx->copy_stream) cudaStreamSynchronize(ctx->copy_stream);
        if (ctx->aux_stream) cudaStreamSynchronize(ctx->aux_stream);
        reclaim(ctx, true);
        cache_drain(ctx);
        cudaStreamSynchronize(ctx->stream);
        if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
        if (ctx->aux_stream) cudaStreamDestroy(ctx->aux_stream);
        if (ctx->h2d_stream) {
            cudaStreamSynchronize(ctx->h2d_stream);
            cudaStreamDestroy(ctx->h2d_stream);
        }
        for (auto& e : ctx->h2d_done)
            if (e) cudaEventDestroy(e);
        for (auto& e : ctx->d2h_done)
            if (e) cudaEventDestroy(e);
        for (auto& s : ctx->stages) {
            cudaEventDestroy(s.a);
            cudaEventDestroy(s.b);
        }
        if (ctx->pinned_scratch) cudaFreeHost(ctx->pinned_scratch);
        if (ctx->sync_ev) cudaEventDestroy(ctx->sync_ev);
        if (ctx->arena) cudaFree(ctx->arena);
        if (ctx->hilbert3) cudaFree(ctx->hilbert3);
        if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
        delete ctx;
    });
}

int lo_context_synchronize(lo_context* ctx) {
    return api_ctx(ctx, [&] {
        sync(ctx);
        LO_CUDA(cudaStreamSynchronize(ctx->copy_stream));
        LO_CUDA(cudaStreamSynchronize(ctx->h2d_stream));
        LO_CUDA(cudaStreamSynchronize(ctx->aux_stream));
        reclaim(ctx, true);  // parked large buffers stay parked (bounded; LO_OPT_RELEASE_SCRATCH frees them)
    });
}
void* lo_context_stream(lo_context* ctx) { return ctx ? ctx->stream : nullptr; }

int lo_context_join(lo_context* ctx) {
    return api_ctx(ctx, [&] {
        for (cudaStream_t s : {ctx->aux_stream, ctx->copy_stream}) {
            cudaEvent_t ev;
            LO_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            LO_CUDA(cudaEventRecord(ev, s));
            LO_CUDA(cudaStreamWaitEvent(ctx->stream, ev, 0));
            cudaEventDestroy(ev);
        }
    });
}

int lo_context_set_option(lo_context* ctx, int option, int64_t value) {
    return api_ctx(ctx, [&] {
        switch (option) {
            case LO_OPT_CENTRE_ORDER: ctx->centre_sort = value != 0; break;
            case LO_OPT_RELEASE_SCRATCH:
                if (value) {
                    sync(ctx);
                    if (ctx->arena) cudaFree(ctx->arena);
                    ctx->arena = nullptr;
                    ctx->arena_bytes = 0;
                    ctx->arena_budgeted = 0;
                    cache_drain(ctx);
                    sync(ctx);
                }
                break;
            default: throw Error(LO_INVALID_ARGUMENT, "unknown context option");
        }
    });
}

int lo_context_set_timing(lo_context* ctx, int enabled) {
    return api_ctx(ctx, [&] {
        ctx->timing = enabled != 0;
        ctx->stage_ms.clear();
    });
}

int lo_context_stage_times(lo_context* ctx, char* names, int name_len, double* ms, int cap) {
    int n = 0;
    const int rc = api_ctx(ctx, [&] {
        resolve_stages(ctx);
        for (auto& [name, t] : ctx->stage_ms) {
            if (n >= cap) break;
            if (names && name_len > 0) {
                std::strncpy(names + static_cast<size_t>(n) * name_len, name.c_str(), name_len - 1);
                names[static_cast<size_t>(n) * name_len + name_len - 1] = 0;
            }
            if (ms) ms[n] = t;
            ++n;
        }
        ctx->stage_ms.clear();
    });
    return rc == LO_OK ? n : -rc;
}

int lo_device_alloc(lo_context* ctx, uint64_t bytes, void** out_dev) {
    return api_ctx(ctx, [&] {
        *out_dev = dalloc(ctx, bytes);
        sync(ctx);
    });
}
int lo_device_free(lo_context* ctx, void* dev) {
    return api_ctx(ctx, [&] {
        dfree(ctx, dev);
        sync(ctx);
    });
}
int lo_memcpy_h2d(lo_context* ctx, void* dst, const void* src, uint64_t bytes) {
    return api_ctx(ctx, [&] {
        LO_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
        sync(ctx);
    });
}
int lo_h2d_begin(lo_context* ctx, void* dst, const void* src, uint64_t bytes, int slot) {
    return api_ctx(ctx, [&] {
        require(slot >= 0 && slot < lo_context::kH2dSlots, LO_INVALID_ARGUMENT, "h2d slot out of range");
        LO_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->h2d_stream));
        LO_CUDA(cudaEventRecord(ctx->h2d_done[slot], ctx->h2d_stream));
    });
}
int lo_h2d_wait(lo_context* ctx, int slot) {
    return api_ctx(ctx, [&] {
        require(slot >= 0 && slot < lo_context::kH2dSlots, LO_INVALID_ARGUMENT, "h2d slot out of range");
        LO_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->h2d_done[slot], 0));
    });
}
int lo_d2h_fence(lo_context* ctx, int slot) {
    return api_ctx(ctx, [&] {
        require(slot >= 0 && slot < lo_context::kH2dSlots, LO_INVALID_ARGUMENT, "d2h slot out of range");
        LO_CUDA(cudaEventRecord(ctx->d2h_done[slot], ctx->copy_stream));
    });
}
int lo_d2h_wait(lo_context* ctx, int slot) {
    return api_ctx(ctx, [&] {
        require(slot >= 0 && slot < lo_context::kH2dSlots, LO_INVALID_ARGUMENT, "d2h slot out of range");
        spin_wait(ctx->d2h_done[slot]);
        reclaim(ctx, false);
    });
}
int lo_memcpy_d2h(lo_context* ctx, void* dst, const void* src, uint64_t bytes) {
    return api_ctx(ctx, [&] {
        LO_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        sync(ctx);
    });
}
int lo_host_alloc_pinned(uint64_t bytes, void** out_host) {
    return api([&] { LO_CUDA(cudaMallocHost(out_host, bytes)); });
}
int lo_host_free_pinned(void* host) { return api([&] { LO_CUDA(cudaFreeHost(host)); }); }

int lo_flush_l2(lo_context* ctx, void* scratch, uint64_t bytes) {
    return api_ctx(ctx, [&] { LO_CUDA(cudaMemsetAsync(scratch, 0x5a, bytes, ctx->stream)); });
}

}  // extern "C"
