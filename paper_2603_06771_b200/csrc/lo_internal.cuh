// lo_internal.cuh -- shared types and device helpers of the B200 path (sm_100a only).
//
// Everything FP64 here is compiled with -fmad=false so the device evaluates exactly the
// reference's expression trees: ((dx*dx + dy*dy) + dz*dz) with
// no DFMA contraction.
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <stdexcept>
#include <string>
#include <atomic>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "../../include/linoct_b200.h"

namespace lo {

using u8 = std::uint8_t;
using u16 = std::uint16_t;
using u32 = std::uint32_t;
using u64 = std::uint64_t;
using i32 = std::int32_t;
using i64 = std::int64_t;

constexpr int kMaxLevel = 21;

// ---- errors ---------------------------------------------------------------------------
struct Error : std::runtime_error {
    int status;
    Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};
[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file, int line);
#define LO_CUDA(call)                                                          \
    do {                                                                       \
        cudaError_t e_ = (call);                                               \
        if (e_ != cudaSuccess) ::lo::throw_cuda(e_, #call, __FILE__, __LINE__); \
    } while (0)
// Every kernel launch is followed by exactly one LO_CHECK_LAUNCH(), which also counts it
// (lo_launch_count(): the harness's evidence of how many of our kernels ran).
void count_launch();
#define LO_CHECK_LAUNCH()                 \
    do {                                  \
        LO_CUDA(cudaGetLastError());      \
        ::lo::count_launch();             \
    } while (0)

inline void require(bool ok, int status, const std::string& msg) {
    if (!ok) throw Error(status, msg);
}
// literal messages: no std::string is built unless the check fails (hot host loops)
inline void require(bool ok, int status, const char* msg) {
    if (!ok) throw Error(status, msg);
}

// ---- curve tables (CurveStepper, sfc.hpp:143-164) -----------------------------------------
// enc[s*8 + g] = (code digit c) | (next state << 3) for octant digit g = x<<2|y<<1|z;
// dec[s*8 + c] = (octant digit g) | (next state << 3).  Morton has 1 state, Hilbert 24.
struct CurveTables {
    u8 enc[32 * 8];
    u8 dec[32 * 8];
    int states;
};
const CurveTables& curve_tables(int curve);  // host-derived once from the codec (tables.cpp)

// ---- device-side handles ----------------------------------------------------------------
// Traversal node: non-empty octree nodes in a children-contiguous layout (root = 0).  The
// box is the exact (tight) min/max of the node's points: any box that contains a node's
// points gives the reference's result sets under exact non-FMA arithmetic.
struct __align__(16) TNode {
    double lo[3];
    double hi[3];
    u32 begin, end;    // sorted-cloud index range [begin, end)
    u32 child0;        // first child tnode (children contiguous, code order)
    u32 nchild;        // 0 for a leaf
};
static_assert(sizeof(TNode) == 64, "TNode must be 64 bytes");

// FP32 shadow of a TNode for the filtered search: the box relative to the cloud origin,
// rounded outward (directed rounding), so it still contains every point's exact relative
// position.  a = (lo.xyz, begin bits), b = (hi.xyz, end bits), c = (child0, nchild, -, -).
struct __align__(16) TNodeF {
    float4 a;
    float4 b;
    uint4 c;
};
static_assert(sizeof(TNodeF) == 48, "TNodeF must be 48 bytes");

}  // namespace lo

struct lo_context {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    bool timing = false;
    int sm_count = 148;
    struct Stage {
        std::string name;
        cudaEvent_t a, b;
    };
    std::vector<Stage> stages;          // pending stage events (resolved on query)
    std::vector<std::pair<std::string, float>> stage_ms;
    void* pinned_scratch = nullptr;     // small mapped pinned buffer for scalar reads
    void* pinned_scratch_dev = nullptr; // its device alias
    void* arena = nullptr;              // persistent device scratch (radius records)
    size_t arena_bytes = 0;
    uint64_t arena_budgeted = 0;  // record demand (bytes) the arena was last sized for under the free-memory cap
    // asynchronous result downloads (lo_csr_download_async): D2H on a second stream so the
    // next batch computes while the previous one's results travel; buffers of results destroyed
    // while their copy is in flight are released once the copy has completed.
    cudaStream_t copy_stream = nullptr;
    struct Deferred {
        cudaEvent_t done;
        std::vector<void*> ptrs;
    };
    std::vector<Deferred> deferred;
    // staged input uploads (lo_h2d_begin / lo_h2d_wait): their own stream so an upload for the
    // next batch overlaps this batch's kernels and the D2H copies; one event per slot
    cudaStream_t h2d_stream = nullptr;
    // row digests run here, behind the fill, so the caller's next batch can start its count pass
    cudaStream_t aux_stream = nullptr;
    // large result buffers released while another stream may still read them are parked here
    // with an event and reused (or freed) once it has completed -- the stream-ordered pool
    // handles cross-stream frees of multi-GB buffers badly (it grows instead of reusing)
    struct Cached {
        void* p;
        size_t bytes;
        cudaEvent_t ready;
    };
    std::vector<Cached> cache;
    std::unordered_map<void*, size_t> big;  // live buffers handed out from (and parked back to) the cache
    size_t cache_cap = 0;                   // parked-bytes cap (a quarter of the device memory)
    cudaEvent_t sync_ev = nullptr;          // sync(): recorded, then spun on (no sleeping wait)
    static constexpr int kH2dSlots = 4;
    cudaEvent_t h2d_done[kH2dSlots] = {};
    cudaEvent_t d2h_done[kH2dSlots] = {};  // lo_d2h_fence / lo_d2h_wait
    // calls on one context are serialized; built handles stay safe to query from
    // any thread
    std::recursive_mutex mu;
    // handles (coded, octree, csr, knn) that still point here: destroying the context first is a
    // LO_LOGIC_ERROR instead of a use-after-free in their destroy calls
    std::atomic<int> live_handles{0};
    // kernels whose dynamic shared-memory limit was raised on this context's device (function
    // attributes are per device; the flag lives under the context lock)
    unsigned smem_attrs = 0;
    void* hilbert3 = nullptr;  // three-level Hilbert encode table on this device (reorder.cu)
    bool centre_sort = true;   // LO_OPT_CENTRE_ORDER: search explicit centre lists in curve order
};

namespace lo {
// A handle's owning context, counted in lo_context::live_handles while it is set.
class CtxRef {
  public:
    CtxRef() = default;
    CtxRef(const CtxRef&) = delete;
    CtxRef& operator=(const CtxRef&) = delete;
    ~CtxRef() { reset(nullptr); }
    CtxRef& operator=(lo_context* c) {
        reset(c);
        return *this;
    }
    operator lo_context*() const { return p_; }
    lo_context* operator->() const { return p_; }

  private:
    void reset(lo_context* c) {
        if (p_) p_->live_handles.fetch_sub(1);
        p_ = c;
        if (p_) p_->live_handles.fetch_add(1);
    }
    lo_context* p_ = nullptr;
};
}  // namespace lo

struct lo_coded {
    lo::CtxRef ctx;
    std::mutex lazy_mu;  // lazily built device data (ensure_float_shadows) is published under it
    lo::u64 n = 0;
    int curve = 0, level = lo::kMaxLevel;
    double disc_box[6] = {};
    double cloud_box[6] = {};
    double scale[3] = {};
    double *x = nullptr, *y = nullptr, *z = nullptr;  // sorted SoA coordinates
    lo::u64* codes = nullptr;                         // sorted codes
    lo::u32* perm = nullptr;                          // perm[new] = old
    // FP32 filter copy: fl32(fl64(p - origin)), origin = disc box min (search_common.cuh)
    float4* pf = nullptr;
    double origin[3] = {};
    double bmax = 0.0;  // >= |p - origin| on every axis (the cube side)
    cudaEvent_t reader = nullptr;  // another stream (broadcast / peer copy) reads the buffers
};

struct lo_octree {
    lo::CtxRef ctx;
    std::mutex lazy_mu;  // lazily built tf / rb / rbf are published under it, complete
    const lo_coded* coded = nullptr;
    lo::u64 points = 0, leaves = 0, internal = 0, tnodes = 0;
    lo::i32 root = 0;
    lo::u32 n_max = 0;
    int level = lo::kMaxLevel, curve = 0;
    double disc_box[6] = {};
    lo::u64* bounds = nullptr;          // [leaves+1]
    lo::u32* offsets = nullptr;         // [leaves+1]
    lo_internal_node* nodes = nullptr;  // [internal]
    lo::TNode* tn = nullptr;            // [tnodes]
    lo::TNodeF* tf = nullptr;           // [tnodes] FP32 shadow (built lazily for replicas)
    double* rb = nullptr;               // [tnodes*6] padded octant boxes (Struct; built lazily)
    float4* rbf = nullptr;              // [tnodes*2] the same, FP32 outward-rounded, relative to origin
    int max_depth = 0;
    cudaEvent_t reader = nullptr;       // another stream (broadcast / peer copy) reads the buffers
};

namespace lo {
// Lazily (re)build the FP32 shadows (after a broadcast the replicas only hold the exact data).
void ensure_float_shadows(lo_context* ctx, const lo_coded* coded, const lo_octree* tree);
// Lazily build the reference's padded octant box of every traversal node (octant_bounds,
// sfc.cpp:110-127), which decides neighbours_struct's Contains / Disjoint (search.cpp:92-96).
void ensure_ref_boxes(lo_context* ctx, const lo_coded* coded, const lo_octree* tree);
}  // namespace lo

struct lo_csr {
    lo::CtxRef ctx;
    lo::u64 rows = 0, total = 0;
    double mean = 0.0;
    float ms = 0.f;
    lo::u64* offsets = nullptr;   // [rows+1]
    lo::u32* indices = nullptr;   // [total]
    lo::u32* counts = nullptr;    // [rows]
    lo::u64* fps = nullptr;       // [rows] or null
    // RadiusMethod::Struct (RangedResult, search.hpp:18-56): per row the coalesced contained
    // ranges (begin, end) and the individually tested singles; `indices` is the expansion,
    // materialised on demand.
    bool is_struct = false;
    lo::u64 total_ranges = 0, total_singles = 0;
    lo::u64* range_offsets = nullptr;   // [rows+1]
    lo::u32* ranges = nullptr;          // [2*total_ranges]
    lo::u64* single_offsets = nullptr;  // [rows+1]
    lo::u32* singles = nullptr;         // [total_singles]
    cudaEvent_t copied = nullptr;       // last lo_csr_download_async (null: none pending)
    cudaEvent_t digested = nullptr;     // digests computed on the aux stream (null: inline / none)
    unsigned copy_mask = 0;             // buffers it reads: 1 counts, 2 fps, 4 offsets, 8 indices
    // block sizes of counts / fps / offsets / indices when they came from big_alloc (0: dalloc)
    size_t cap[4] = {0, 0, 0, 0};
};

namespace lo {
struct Queries;
// radius_struct.cu: RadiusMethod::Struct batch, the on-demand expansion, buffer release.
lo_csr* radius_struct_search(lo_context* ctx, const lo_octree* t, const lo_coded* c, int shape,
                             double r, const Queries& q, bool fingerprint);
void ensure_expanded(lo_context* ctx, lo_csr* csr);
// centres.cu: explicit centre lists searched in curve order (sorted), rows scattered back.
struct SortedCentres {
    u32* idx = nullptr;  // ascending centre indices
    u32* pos = nullptr;  // their positions in the caller's list
};
SortedCentres sort_centres(lo_context* ctx, const u32* centres, u64 m);
void unsort_csr(lo_context* ctx, const SortedCentres& s, lo_csr* c);
void unsort_knn(lo_context* ctx, const SortedCentres& s, lo_knn_result* r);
// reorder.cu: stable LSD sort of u64 keys (passes for `level`*3 bits, constant digits skipped
// per hist_host[8*256]); perm = original positions.
// hist_dev (optional): the same histogram on the device -- the digit bases are then scanned there
// instead of uploaded (no host->device copy that could queue behind a pending upload).
void radix_sort(lo_context* ctx, u64* keys, u64 n, const u32* hist_host, int level, u64* keys_sorted, u32* perm,
                const u32* hist_dev = nullptr);
// reorder.cu: positions of arbitrary query points (SoA, device) in curve order.
u32* sort_points_sfc(lo_context* ctx, const lo_coded* c, const double* x, const double* y, const double* z,
                     u64 m);
// centres.cu: gather query arrays (x, y, z, f) into curve order in place.
void gather_queries(lo_context* ctx, const u32* pos, u64 m, double*& x, double*& y, double*& z, float4*& f);
// reorder.cu: reorder_cloud over a device AoS cloud.
lo_coded* reorder_device(lo_context* ctx, const double* xyz, u64 n, int curve, int level);
// octree.cu: LinearOctree(LeafArray, Discretizer, Curve, n_max) over host leaf arrays.
lo_octree* octree_from_leaves(lo_context* ctx, const lo_coded* coded, const u64* b_host,
                              const u32* off_host, u64 count, const double disc_box[6], int level,
                              int curve, u32 n_max);
void free_csr_buffers(lo_context* ctx, lo_csr* csr);
}  // namespace lo

struct lo_knn_result {
    lo::CtxRef ctx;
    lo::u64 rows = 0;
    lo::u32 k = 0, keff = 0;
    float ms = 0.f;
    lo::u32* idx = nullptr;      // [rows*keff]
    double* dist = nullptr;      // [rows*keff]
    lo::u64* fps = nullptr;      // [rows] or null
    cudaEvent_t copied = nullptr; // last lo_knn_download_async (null: none pending)
};

namespace lo {

// ---- memory + timing helpers (context.cu) ------------------------------------------------
void* dalloc(lo_context* ctx, size_t bytes);
// Large buffers through the context's cache: reuse a parked buffer whose last reader finished,
// else allocate; release parks it behind an event recorded on `last_use`.
void* big_alloc(lo_context* ctx, size_t bytes, size_t* got);
template <class T>
T* big_alloc_t(lo_context* ctx, u64 n, size_t* got) {
    return static_cast<T*>(big_alloc(ctx, n ? n * sizeof(T) : 16, got));
}
void big_release(lo_context* ctx, void* p, size_t bytes, cudaStream_t last_use);
void cache_drain(lo_context* ctx);
// Releases deferred buffers whose async copies finished (all of them when wait is true).
void reclaim(lo_context* ctx, bool wait);
void dfree(lo_context* ctx, void* p);
template <class T>
T* dalloc_t(lo_context* ctx, size_t count) {
    return static_cast<T*>(dalloc(ctx, count * sizeof(T) + (count == 0)));
}
// Persistent per-context scratch of at least `bytes` (grown on demand, reused across calls,
// released with the context).  Throws LO_OUT_OF_MEMORY when it cannot grow.
void* arena(lo_context* ctx, size_t bytes);
void stage_begin(lo_context* ctx, const char* name);
void stage_end(lo_context* ctx);
void sync(lo_context* ctx);
void spin_wait(cudaEvent_t ev);  // busy-waits for a recorded event
// Copies `bytes` (<= 16384, 4-byte aligned) of device memory into ctx->pinned_scratch and waits.
// A one-warp kernel stores them through the mapped alias instead of a cudaMemcpy: a D2H copy on
// the context stream queued behind the copy engine's pending result downloads (lo_csr_download_async
// of the previous batch) and stalled every batch by the length of that download.
void fetch_small(lo_context* ctx, const void* dev, size_t bytes);
template <class T>
T read_scalar(lo_context* ctx, const T* dev) {
    fetch_small(ctx, dev, sizeof(T));
    T v;
    std::memcpy(&v, ctx->pinned_scratch, sizeof(T));
    return v;
}

// scan.cu: exclusive scan, out has n+1 entries (out[n] = total)
void exclusive_scan_u32_to_u64(lo_context* ctx, const u32* in, u64* out, u64 n);
void exclusive_scan_u32(lo_context* ctx, const u32* in, u32* out, u64 n);

// ---- device helpers ---------------------------------------------------------------------
__host__ __device__ inline u64 spread3(u64 v) {
    v &= 0x1fffffULL;
    v = (v | v << 32) & 0x001f00000000ffffULL;
    v = (v | v << 16) & 0x001f0000ff0000ffULL;
    v = (v | v << 8) & 0x100f00f00f00f00fULL;
    v = (v | v << 4) & 0x10c30c30c30c30c3ULL;
    v = (v | v << 2) & 0x1249249249249249ULL;
    return v;
}
__host__ __device__ inline u32 compact3(u64 v) {
    v &= 0x1249249249249249ULL;
    v = (v ^ (v >> 2)) & 0x10c30c30c30c30c3ULL;
    v = (v ^ (v >> 4)) & 0x100f00f00f00f00fULL;
    v = (v ^ (v >> 8)) & 0x001f0000ff0000ffULL;
    v = (v ^ (v >> 16)) & 0x001f00000000ffffULL;
    v = (v ^ (v >> 32)) & 0x1fffffULL;
    return static_cast<u32>(v);
}

// Order-preserving integer image of a double (exact min/max via integer atomics).
__host__ __device__ inline u64 dbl_order_key(double v) {
#ifdef __CUDA_ARCH__
    const u64 u = static_cast<u64>(__double_as_longlong(v));
#else
    u64 u;
    std::memcpy(&u, &v, 8);
#endif
    return (u & 0x8000000000000000ULL) ? ~u : (u | 0x8000000000000000ULL);
}
__host__ __device__ inline double dbl_from_order_key(u64 k) {
    const u64 u = (k & 0x8000000000000000ULL) ? (k & 0x7fffffffffffffffULL) : ~k;
#ifdef __CUDA_ARCH__
    return __longlong_as_double(static_cast<long long>(u));
#else
    double v;
    std::memcpy(&v, &u, 8);
    return v;
#endif
}

// FNV-1a-64 of a u32 index widened to u64 (search.cpp:263-271): the 4 zero high bytes only
// multiply, so they fold into one multiplication by prime^5 after the 4th byte.
__device__ __forceinline__ u64 fnv_u32(u64 h, u32 v) {
    constexpr u64 P = 0x100000001b3ULL;
    constexpr u64 P5 = P * P * P * P * P;
    h ^= v & 0xffu;
    h *= P;
    h ^= (v >> 8) & 0xffu;
    h *= P;
    h ^= (v >> 16) & 0xffu;
    h *= P;
    h ^= v >> 24;
    h *= P5;
    return h;
}
// The same for an index known to be < 2^24 (clouds of at most 16.7M points): its fourth byte is
// zero as well, so five zero bytes fold into prime^6 (two fewer integer ops per index).
__device__ __forceinline__ u64 fnv_u24(u64 h, u32 v) {
    constexpr u64 P = 0x100000001b3ULL;
    constexpr u64 P6 = P * P * P * P * P * P;
    h ^= v & 0xffu;
    h *= P;
    h ^= (v >> 8) & 0xffu;
    h *= P;
    h ^= v >> 16;
    h *= P6;
    return h;
}
__device__ __forceinline__ u64 fnv_u64(u64 h, u64 v) {
    constexpr u64 P = 0x100000001b3ULL;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        h ^= (v >> (8 * i)) & 0xffu;
        h *= P;
    }
    return h;
}
constexpr u64 kFnvOffset = 0xcbf29ce484222325ULL;

void set_last_error(const char* msg);

// Runs an API body, mapping exceptions to status codes (no exception crosses the C ABI).
template <class F>
int api(F&& f) {
    try {
        f();
        return LO_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.status;
    } catch (const std::bad_alloc&) {
        set_last_error("host allocation failed");
        return LO_OUT_OF_MEMORY;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return LO_LOGIC_ERROR;
    }
}

// Makes `device` current for the scope (a context may be used from any host thread, whose
// current device can be another one) and restores the caller's device afterwards.
class DeviceGuard {
  public:
    explicit DeviceGuard(int device) {
        if (cudaGetDevice(&prev_) != cudaSuccess) {
            cudaGetLastError();
            prev_ = -1;
        }
        if (prev_ != device) {
            cudaSetDevice(device);
        } else {
            prev_ = -1;
        }
    }
    ~DeviceGuard() {
        if (prev_ >= 0) cudaSetDevice(prev_);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;

  private:
    int prev_ = -1;
};

// api() under the context's lock, on the context's device.
template <class F>
int api_ctx(lo_context* ctx, F&& f) {
    if (!ctx) return api([] { throw Error(LO_INVALID_ARGUMENT, "null context"); });
    std::lock_guard<std::recursive_mutex> lock(ctx->mu);
    DeviceGuard dev(ctx->device);
    return api(std::forward<F>(f));
}

// Raises a kernel's dynamic shared-memory limit once per context (= per device).
enum : unsigned { kAttrSort = 1u, kAttrReplay = 2u, kAttrKnnW1 = 4u, kAttrKnnW2 = 8u };
template <class K>
void ensure_smem_attr(lo_context* ctx, unsigned bit, K kernel, size_t smem) {
    if (ctx->smem_attrs & bit) return;
    LO_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    ctx->smem_attrs |= bit;
}

inline int ceil_div(u64 a, u64 b) { return static_cast<int>((a + b - 1) / b); }

// Test knobs, read on every call (not cached) so a test can flip them between calls:
//   LO_FORCE_FP64=1      every search takes its exact FP64 kernel (the FP32 filter off), the path
//                        radii below ~2.4e-5 x the cube side take on their own
//   LO_RADIUS_NO_FUSE=1  radius fill by a second walk instead of replaying count-pass records
//   LO_REC_CAP=<n>       records per tile before a tile overflows to the fill walk (default 128)
//   LO_KNN_SELECT=1      kNN by candidate collection + warp selection (knn_select.cuh), with
//                        LO_KNN_WIN / LO_KNN_CAP / LO_KNN_LIST_MB (bound window, list capacity, chunk)
//   LO_KNN_WARP=1        kNN by the warp-cooperative heaps (knn_warp.cuh)
// Diagnostics (read once): LO_DEBUG=1 (arena growth, record overflow, kNN select chunks),
// LO_DEBUG_ALLOC=1 (slow cudaMallocAsync calls), LO_DEBUG_HOST=1 (host calls over 1 ms, and the host
// segments of every radius call).
inline bool env_flag(const char* name) {
    const char* e = std::getenv(name);
    return e && *e && *e != '0';
}
inline bool force_fp64() { return env_flag("LO_FORCE_FP64"); }

// LO_DEBUG_HOST=1 (diagnostic): host calls of the library that take over 1 ms are logged to stderr
struct SlowLog {
    const char* what;
    size_t arg;
    std::chrono::steady_clock::time_point t0;
    static bool on() {
        static const bool enabled = std::getenv("LO_DEBUG_HOST") != nullptr;
        return enabled;
    }
    SlowLog(const char* w, size_t a) : what(w), arg(a) {
        if (on()) t0 = std::chrono::steady_clock::now();
    }
    ~SlowLog() {
        if (!on()) return;
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (ms > 1.0) std::fprintf(stderr, "[lo] slow host call %s(%zu): %.2f ms\n", what, arg, ms);
    }
};

}  // namespace lo
