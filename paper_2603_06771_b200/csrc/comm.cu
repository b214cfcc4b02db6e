// comm.cu -- multi-GPU in the C ABI: one process per GPU, an NCCL communicator
// per context, the structure built once and broadcast over NVLink / NVSwitch, queries sharded
// by contiguous SFC ranges, CSR rows concatenated by offset.
//
// The reference's parallel loop (search.cpp:297, OpenMP over centres) becomes a loop over GPUs:
// rank r owns the centres [n*r/G, n*(r+1)/G) of the sorted cloud.  Queries are independent and
// the structure is read-only, so the only exchanges are the structure broadcast and one
// all-gather of the per-rank neighbour totals (the global row base of each rank's CSR shard).
//
// NCCL is loaded with dlopen at lo_comm_init (the process's libnccl.so.2 -- torch's, when it is
// already loaded -- else the system one), so the library has no link-time NCCL dependency and
// single-GPU callers never touch it.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "lo_internal.cuh"

struct lo_comm {
    lo::CtxRef ctx;
    ncclComm_t nccl = nullptr;
    int rank = 0, nranks = 1;
    cudaStream_t stream = nullptr;  // broadcasts / all-gathers overlap the context stream's work
    cudaEvent_t done = nullptr;     // last collective enqueued on `stream`
};

namespace lo {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    std::string error;
};

static const NcclApi& nccl_api() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.error = std::string("NCCL not available: ") + dlerror();
            return;
        }
        auto sym = [&](const char* name) {
            void* p = dlsym(h, name);
            if (!p && api.error.empty()) api.error = std::string("NCCL symbol missing: ") + name;
            return p;
        };
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
        api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(sym("ncclBroadcast"));
        api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    });
    require(api.error.empty(), LO_NCCL_ERROR, api.error);
    return api;
}

static void nccl_check(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return;
    const NcclApi& a = nccl_api();
    throw Error(LO_NCCL_ERROR, std::string(what) + ": " + (a.GetErrorString ? a.GetErrorString(r) : "NCCL error"));
}
#define LO_NCCL(call) nccl_check((call), #call)

// Contiguous, balanced split of [0, n): rank r owns [n*r/G, n*(r+1)/G).
static void shard(u64 n, int rank, int nranks, u64* b, u64* e) {
    *b = static_cast<u64>((static_cast<unsigned __int128>(n) * rank) / nranks);
    *e = static_cast<u64>((static_cast<unsigned __int128>(n) * (rank + 1)) / nranks);
}

// Makes `s` wait for everything enqueued so far on `after`.
static void stream_after(cudaStream_t s, cudaStream_t after) {
    cudaEvent_t ev;
    LO_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    LO_CUDA(cudaEventRecord(ev, after));
    LO_CUDA(cudaStreamWaitEvent(s, ev, 0));
    cudaEventDestroy(ev);  // released once the recorded work completes
}

// A handle's buffers are read by another stream (a broadcast or a peer copy): its destroy orders
// the frees behind `ev` (lo_coded_destroy / lo_octree_destroy wait on `reader`).
static void mark_reader(cudaEvent_t& reader, cudaStream_t s) {
    if (!reader) LO_CUDA(cudaEventCreateWithFlags(&reader, cudaEventDisableTiming));
    LO_CUDA(cudaEventRecord(reader, s));
}

struct StructHeader {
    lo_coded_info ci;
    lo_octree_info ti;
};

struct Buf {
    void* p;
    size_t bytes;
};

static std::vector<Buf> coded_bufs(const lo_coded* c) {
    return {{c->x, 8 * c->n}, {c->y, 8 * c->n}, {c->z, 8 * c->n}, {c->codes, 8 * c->n}, {c->perm, 4 * c->n}};
}
static std::vector<Buf> tree_bufs(const lo_octree* t) {
    return {{t->bounds, 8 * (t->leaves + 1)},
            {t->offsets, 4 * (t->leaves + 1)},
            {t->nodes, sizeof(lo_internal_node) * t->internal},
            {t->tn, sizeof(TNode) * t->tnodes}};
}

static StructHeader header_of(const lo_coded* c, const lo_octree* t) {
    StructHeader h{};
    require(lo_coded_info_get(c, &h.ci) == LO_OK && lo_octree_info_get(t, &h.ti) == LO_OK, LO_INVALID_ARGUMENT,
            "broadcast: bad root handles");
    return h;
}

// Empty handles of the header's shape on ctx (lo_coded_create_empty / lo_octree_create_empty).
static void create_empty(lo_context* ctx, const StructHeader& h, lo_coded** c, lo_octree** t) {
    if (lo_coded_create_empty(ctx, &h.ci, c) != LO_OK) throw Error(LO_OUT_OF_MEMORY, lo_last_error());
    if (lo_octree_create_empty(ctx, *c, &h.ti, t) != LO_OK) {
        const std::string m = lo_last_error();
        lo_coded_destroy(*c);
        *c = nullptr;
        throw Error(LO_OUT_OF_MEMORY, m);
    }
}

}  // namespace lo

using namespace lo;

extern "C" {

int lo_shard_range(uint64_t n, int rank, int nranks, uint64_t* begin, uint64_t* end) {
    return api([&] {
        require(nranks >= 1 && rank >= 0 && rank < nranks && begin && end, LO_INVALID_ARGUMENT,
                "shard: rank out of range");
        shard(n, rank, nranks, begin, end);
    });
}

int lo_comm_unique_id(void* id_out) {
    return api([&] {
        require(id_out != nullptr, LO_INVALID_ARGUMENT, "null id buffer");
        ncclUniqueId id;
        LO_NCCL(nccl_api().GetUniqueId(&id));
        std::memcpy(id_out, &id, sizeof id);
    });
}

int lo_comm_init(lo_context* ctx, const void* id, int nranks, int rank, lo_comm** out) {
    return api_ctx(ctx, [&] {
        require(id && out && nranks >= 1 && rank >= 0 && rank < nranks, LO_INVALID_ARGUMENT,
                "comm: bad rank / size");
        static_assert(sizeof(ncclUniqueId) == LO_COMM_ID_BYTES, "NCCL unique id size");
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof uid);
        auto* c = new lo_comm;
        c->ctx = ctx;
        c->rank = rank;
        c->nranks = nranks;
        try {
            LO_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
            LO_CUDA(cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming));
            LO_NCCL(nccl_api().CommInitRank(&c->nccl, nranks, uid, rank));
        } catch (...) {
            if (c->stream) cudaStreamDestroy(c->stream);
            if (c->done) cudaEventDestroy(c->done);
            delete c;
            throw;
        }
        *out = c;
    });
}

int lo_comm_info(const lo_comm* comm, int* rank, int* nranks) {
    return api([&] {
        require(comm != nullptr, LO_INVALID_ARGUMENT, "null comm");
        if (rank) *rank = comm->rank;
        if (nranks) *nranks = comm->nranks;
    });
}

int lo_comm_destroy(lo_comm* comm) {
    if (!comm) return LO_OK;
    return api_ctx(comm->ctx, [&] {
        cudaStreamSynchronize(comm->stream);
        if (comm->nccl) nccl_api().CommDestroy(comm->nccl);
        cudaStreamDestroy(comm->stream);
        cudaEventDestroy(comm->done);
        delete comm;
    });
}

int lo_broadcast_structure(lo_comm* comm, const lo_coded* coded, const lo_octree* tree, int root,
                           lo_coded** coded_out, lo_octree** tree_out) {
    if (!comm) return api([] { throw Error(LO_INVALID_ARGUMENT, "null comm"); });
    return api_ctx(comm->ctx, [&] {
        lo_context* ctx = comm->ctx;
        const NcclApi& nc = nccl_api();
        require(root >= 0 && root < comm->nranks, LO_INVALID_ARGUMENT, "broadcast: root out of range");
        const bool is_root = comm->rank == root;
        require(!is_root || (coded && tree && coded->ctx == ctx && tree->ctx == ctx), LO_INVALID_ARGUMENT,
                "broadcast: the root passes its (coded, tree) built on this context");
        require(is_root || (coded_out && tree_out), LO_INVALID_ARGUMENT, "broadcast: null output handles");
        cudaEvent_t t0 = nullptr, t1 = nullptr;
        if (ctx->timing) {
            LO_CUDA(cudaEventCreate(&t0));
            LO_CUDA(cudaEventCreate(&t1));
        }
        // the root's structure is complete on its stream before anything is sent
        stream_after(comm->stream, ctx->stream);
        if (t0) LO_CUDA(cudaEventRecord(t0, comm->stream));
        // 1. the header (sizes): receivers need it on the host to allocate
        StructHeader h = is_root ? header_of(coded, tree) : StructHeader{};
        StructHeader* hd = dalloc_t<StructHeader>(ctx, 1);
        stream_after(comm->stream, ctx->stream);  // the allocation is stream-ordered on ctx->stream
        if (is_root) LO_CUDA(cudaMemcpyAsync(hd, &h, sizeof h, cudaMemcpyHostToDevice, comm->stream));
        LO_NCCL(nc.Broadcast(hd, hd, sizeof h, ncclChar, root, comm->nccl, comm->stream));
        LO_CUDA(cudaMemcpyAsync(&h, hd, sizeof h, cudaMemcpyDeviceToHost, comm->stream));
        LO_CUDA(cudaStreamSynchronize(comm->stream));
        dfree(ctx, hd);
        // 2. receivers allocate empty handles of that shape
        lo_coded* c = const_cast<lo_coded*>(coded);
        lo_octree* t = const_cast<lo_octree*>(tree);
        if (!is_root) create_empty(ctx, h, &c, &t);  // synchronous: buffers exist before the copy
        // 3. every buffer in one NCCL group (NVLink / NVSwitch; NVLS when NCCL picks it)
        try {
            std::vector<Buf> bufs = coded_bufs(c);
            for (const Buf& b : tree_bufs(t)) bufs.push_back(b);
            LO_NCCL(nc.GroupStart());
            for (const Buf& b : bufs)
                if (b.bytes) LO_NCCL(nc.Broadcast(b.p, b.p, b.bytes, ncclChar, root, comm->nccl, comm->stream));
            LO_NCCL(nc.GroupEnd());
            LO_CUDA(cudaEventRecord(comm->done, comm->stream));
            if (t1) {
                LO_CUDA(cudaEventRecord(t1, comm->stream));
                ctx->stages.push_back({"broadcast", t0, t1});
                t0 = t1 = nullptr;
            }
        } catch (...) {
            if (!is_root) {
                lo_octree_destroy(t);
                lo_coded_destroy(c);
            }
            if (t0) cudaEventDestroy(t0);
            if (t1) cudaEventDestroy(t1);
            throw;
        }
        if (is_root) {
            // the root keeps computing (its own shard) while the broadcast runs on the comm stream;
            // destroying its handles orders the frees behind the broadcast
            mark_reader(c->reader, comm->stream);
            mark_reader(t->reader, comm->stream);
            if (coded_out) *coded_out = nullptr;
            if (tree_out) *tree_out = nullptr;
        } else {
            LO_CUDA(cudaStreamWaitEvent(ctx->stream, comm->done, 0));
            ensure_float_shadows(ctx, c, t);  // FP32 filter copies rebuilt locally (not sent)
            *coded_out = c;
            *tree_out = t;
        }
    });
}

int lo_structure_copy(lo_context* dst, const lo_coded* coded, const lo_octree* tree, lo_coded** coded_out,
                      lo_octree** tree_out) {
    return api([&] {
        require(dst && coded && tree && coded_out && tree_out && tree->coded == coded, LO_INVALID_ARGUMENT,
                "structure copy: null handle or tree of another cloud");
        lo_context* src = coded->ctx;
        std::unique_lock<std::recursive_mutex> la(src->mu, std::defer_lock), lb(dst->mu, std::defer_lock);
        if (src == dst) {
            la.lock();
        } else {
            std::lock(la, lb);
        }
        DeviceGuard dev(dst->device);
        StructHeader h = header_of(coded, tree);
        lo_coded* c = nullptr;
        lo_octree* t = nullptr;
        create_empty(dst, h, &c, &t);
        try {
            // the source structure is complete on its stream; copies run on the destination's
            cudaEvent_t ready;
            {
                DeviceGuard sdev(src->device);
                LO_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
                LO_CUDA(cudaEventRecord(ready, src->stream));
            }
            LO_CUDA(cudaStreamWaitEvent(dst->stream, ready, 0));
            cudaEventDestroy(ready);
            std::vector<Buf> from = coded_bufs(coded), to = coded_bufs(c);
            for (const Buf& b : tree_bufs(tree)) from.push_back(b);
            for (const Buf& b : tree_bufs(t)) to.push_back(b);
            stage_begin(dst, "structure_copy");
            for (size_t i = 0; i < from.size(); ++i)
                if (from[i].bytes)
                    LO_CUDA(cudaMemcpyPeerAsync(to[i].p, dst->device, from[i].p, src->device, from[i].bytes,
                                                dst->stream));
            stage_end(dst);
            {
                DeviceGuard sdev(src->device);
                mark_reader(const_cast<lo_coded*>(coded)->reader, dst->stream);
                mark_reader(const_cast<lo_octree*>(tree)->reader, dst->stream);
            }
            ensure_float_shadows(dst, c, t);
        } catch (...) {
            lo_octree_destroy(t);
            lo_coded_destroy(c);
            throw;
        }
        *coded_out = c;
        *tree_out = t;
    });
}

int lo_weighted_bounds(const uint32_t* sample_counts, uint64_t samples, uint32_t stride, uint64_t n,
                       uint32_t base_cost, int nranks, uint64_t* bounds) {
    return api([&] {
        require(bounds && nranks >= 1 && stride >= 1, LO_INVALID_ARGUMENT, "weighted_bounds: bad arguments");
        require(samples == (n + stride - 1) / stride, LO_INVALID_ARGUMENT,
                "weighted_bounds: one sample per stride block expected");
        require(samples == 0 || sample_counts, LO_INVALID_ARGUMENT, "weighted_bounds: null counts");
        // cumulative cost at the end of each stride block (exact in u128 arithmetic)
        std::vector<unsigned __int128> cum(samples);
        unsigned __int128 acc = 0;
        for (u64 j = 0; j < samples; ++j) {
            const u64 q = std::min<u64>(stride, n - j * stride);
            acc += static_cast<unsigned __int128>(q) * (static_cast<u64>(sample_counts[j]) + base_cost);
            cum[j] = acc;
        }
        bounds[0] = 0;
        u64 j = 0;
        for (int r = 1; r < nranks; ++r) {
            const unsigned __int128 target = acc * static_cast<unsigned>(r) / static_cast<unsigned>(nranks);
            while (j < samples && cum[j] <= target) ++j;  // first block whose end passes the target
            // the bound goes to the nearer block edge
            u64 cut = j;
            if (j < samples) {
                const unsigned __int128 before = j ? cum[j - 1] : 0;
                if (target - before > cum[j] - target) cut = j + 1;
            }
            bounds[r] = std::max(bounds[r - 1], std::min<u64>(n, cut * stride));
        }
        bounds[nranks] = n;
    });
}

int lo_radius_work_bounds(lo_context* ctx, const lo_octree* tree, const lo_coded* coded, int shape,
                          double radius, uint32_t stride, int nranks, uint64_t* bounds) {
    return api_ctx(ctx, [&] {
        require(tree && coded && bounds, LO_INVALID_ARGUMENT, "null tree, cloud or bounds");
        require(stride >= 32 && stride % 32 == 0 && nranks >= 1, LO_INVALID_ARGUMENT,
                "radius_work_bounds: stride must be a positive multiple of 32");
        // one whole query tile (32 consecutive centres) at the start of every stride block: sampled
        // tiles stay as compact as the batch's own (every-stride-th centres made each sampled tile
        // span 32 blocks: 6 ms at cfg3 instead of ~1/64 of the count)
        const u64 n = coded->n, samples = (n + stride - 1) / stride;
        std::vector<u32> centres;
        centres.reserve(samples * 32);
        for (u64 j = 0; j < samples; ++j)
            for (u64 i = j * stride; i < std::min<u64>(n, j * stride + 32); ++i) centres.push_back(static_cast<u32>(i));
        std::vector<u32> rows(centres.size()), counts(samples);
        lo_csr* csr = nullptr;
        int rc = lo_radius(ctx, tree, coded, LO_METHOD_LIN, shape, radius, centres.data(), centres.size(), 0, &csr);
        if (rc != LO_OK) throw Error(rc, lo_last_error());
        rc = lo_csr_download(ctx, csr, rows.data(), nullptr, nullptr, nullptr);
        lo_csr_destroy(csr);
        if (rc != LO_OK) throw Error(rc, lo_last_error());
        for (u64 j = 0, c = 0; j < samples; ++j) {  // mean neighbours per query of the sampled tile
            const u64 k = std::min<u64>(32, n - j * stride);
            u64 sum = 0;
            for (u64 i = 0; i < k; ++i) sum += rows[c + i];
            c += k;
            counts[j] = static_cast<u32>((sum + k / 2) / k);
        }
        // per-query fixed cost ~16 neighbour-equivalents (the walk and the tile's buffers)
        rc = lo_weighted_bounds(counts.data(), samples, stride, n, 16, nranks, bounds);
        if (rc != LO_OK) throw Error(rc, lo_last_error());
    });
}

static int radius_sharded_impl(lo_comm* comm, const lo_octree* tree, const lo_coded* coded, int method, int shape,
                               double radius, int fingerprint, const uint64_t* bounds, lo_csr** out,
                               uint64_t* row_begin, uint64_t* row_base, uint64_t* total) {
    if (!comm) return api([] { throw Error(LO_INVALID_ARGUMENT, "null comm"); });
    return api_ctx(comm->ctx, [&] {
        lo_context* ctx = comm->ctx;
        require(tree && coded && out, LO_INVALID_ARGUMENT, "null tree, cloud or output");
        u64 b = 0, e = 0;
        if (bounds) {
            b = bounds[comm->rank];
            e = bounds[comm->rank + 1];
            require(b <= e && e <= coded->n && bounds[0] == 0 && bounds[comm->nranks] == coded->n,
                    LO_INVALID_ARGUMENT, "radius_sharded: bounds must cover [0, n) in order");
        } else {
            shard(coded->n, comm->rank, comm->nranks, &b, &e);
        }
        lo_csr* csr = nullptr;
        const int rc = lo_radius_range(ctx, tree, coded, method, shape, radius, b, e, fingerprint, &csr);
        if (rc != LO_OK) throw Error(rc, lo_last_error());
        // global row base: one all-gather of the per-rank totals (u64: cfg3 exceeds 2^32)
        std::vector<u64> all(comm->nranks, 0);
        u64* d = dalloc_t<u64>(ctx, comm->nranks + 1);
        try {
            LO_CUDA(cudaMemcpyAsync(d + comm->nranks, &csr->total, 8, cudaMemcpyHostToDevice, ctx->stream));
            stream_after(comm->stream, ctx->stream);
            LO_NCCL(nccl_api().AllGather(d + comm->nranks, d, 1, ncclUint64, comm->nccl, comm->stream));
            LO_CUDA(cudaMemcpyAsync(all.data(), d, 8 * comm->nranks, cudaMemcpyDeviceToHost, comm->stream));
            LO_CUDA(cudaStreamSynchronize(comm->stream));
        } catch (...) {
            dfree(ctx, d);
            lo_csr_destroy(csr);
            throw;
        }
        dfree(ctx, d);
        u64 base = 0, sum = 0;
        for (int r = 0; r < comm->nranks; ++r) {
            if (r < comm->rank) base += all[r];
            sum += all[r];
        }
        *out = csr;
        if (row_begin) *row_begin = b;
        if (row_base) *row_base = base;
        if (total) *total = sum;
    });
}

int lo_radius_sharded(lo_comm* comm, const lo_octree* tree, const lo_coded* coded, int method, int shape,
                      double radius, int fingerprint, lo_csr** out, uint64_t* row_begin, uint64_t* row_base,
                      uint64_t* total) {
    return radius_sharded_impl(comm, tree, coded, method, shape, radius, fingerprint, nullptr, out, row_begin,
                               row_base, total);
}

int lo_radius_sharded_bounds(lo_comm* comm, const lo_octree* tree, const lo_coded* coded, int method, int shape,
                             double radius, int fingerprint, const uint64_t* bounds, lo_csr** out,
                             uint64_t* row_begin, uint64_t* row_base, uint64_t* total) {
    if (!bounds) return api([] { throw Error(LO_INVALID_ARGUMENT, "null bounds"); });
    return radius_sharded_impl(comm, tree, coded, method, shape, radius, fingerprint, bounds, out, row_begin,
                               row_base, total);
}

int lo_knn_sharded(lo_comm* comm, const lo_octree* tree, const lo_coded* coded, uint32_t k, int fingerprint,
                   lo_knn_result** out, uint64_t* row_begin) {
    if (!comm) return api([] { throw Error(LO_INVALID_ARGUMENT, "null comm"); });
    return api_ctx(comm->ctx, [&] {
        require(tree && coded && out, LO_INVALID_ARGUMENT, "null tree, cloud or output");
        u64 b = 0, e = 0;
        shard(coded->n, comm->rank, comm->nranks, &b, &e);
        const int rc = lo_knn_range(comm->ctx, tree, coded, k, b, e, fingerprint, out);
        if (rc != LO_OK) throw Error(rc, lo_last_error());
        if (row_begin) *row_begin = b;
    });
}

}  // extern "C"
