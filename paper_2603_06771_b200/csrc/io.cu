// io.cu -- the reference's on-disk formats on the device path:
//   * PCB1 clouds (io.cpp:53-81, :94-106): "PCB1", u64 count, count x (f64 x, y, z), all
//     little-endian.  lo_reorder_pcb streams the file through two pinned staging buffers so
//     the disk read of chunk i+1 overlaps the H2D copy of chunk i, then reorders on the device
//     ("reorder once, store, reuse").  lo_coded_write_pcb stores a sorted cloud.
//   * LOC1 trees (linear_octree.cpp:149-190): "LOC1", u32 level, u32 curve, u32 n_max,
//     6 f64 Discretizer box, u64 count, count u64 boundaries, count u32 offsets.  Loading links
//     the internal nodes on the device from the LeafArray (octree_from_leaves).
// Errors follow the reference: std::runtime_error texts for unreadable / malformed files
// (LO_RUNTIME_ERROR), std::invalid_argument for invalid leaf arrays.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "lo_internal.cuh"

namespace lo {

namespace {

struct File {
    std::FILE* f = nullptr;
    explicit File(std::FILE* p) : f(p) {}
    ~File() {
        if (f) std::fclose(f);
    }
};

// Little-endian wire values (endian.hpp:13-48); the hosts here are little-endian, checked once.
bool host_is_little_endian() {
    const u32 one = 1;
    unsigned char c;
    std::memcpy(&c, &one, 1);
    return c == 1;
}

template <class T>
bool get_le(std::FILE* f, T& v) {
    unsigned char b[sizeof(T)];
    if (std::fread(b, 1, sizeof b, f) != sizeof b) return false;
    u64 u = 0;
    for (int i = static_cast<int>(sizeof(T)) - 1; i >= 0; --i) u = (u << 8) | b[i];
    if constexpr (sizeof(T) == 8) {
        std::memcpy(&v, &u, 8);
    } else {
        const u32 w = static_cast<u32>(u);
        std::memcpy(&v, &w, sizeof(T));
    }
    return true;
}

template <class T>
void put_le(std::FILE* f, T v) {
    u64 u = 0;
    std::memcpy(&u, &v, sizeof(T));
    unsigned char b[sizeof(T)];
    for (int i = 0; i < static_cast<int>(sizeof(T)); ++i) b[i] = static_cast<unsigned char>(u >> (8 * i));
    require(std::fwrite(b, 1, sizeof b, f) == sizeof b, LO_RUNTIME_ERROR, "write failed");
}

constexpr u64 kChunkRecords = 1ull << 21;  // 48 MiB of points per staging buffer

}  // namespace

static lo_coded* reorder_pcb(lo_context* ctx, const char* path, int curve, int level) {
    require(path != nullptr, LO_INVALID_ARGUMENT, "null path");
    require(host_is_little_endian(), LO_RUNTIME_ERROR, "big-endian host");
    const std::string p(path);
    File f(std::fopen(path, "rb"));
    require(f.f != nullptr, LO_RUNTIME_ERROR, "cannot open '" + p + "'");
    char magic[4];
    require(std::fread(magic, 1, 4, f.f) == 4 && std::memcmp(magic, "PCB1", 4) == 0, LO_RUNTIME_ERROR,
            p + ": bad magic at byte offset 0");
    u64 count = 0;
    require(get_le(f.f, count), LO_RUNTIME_ERROR, p + ": truncated count at byte offset 4");
    // a short file fails at its first incomplete record, like the sequential reader (io.cpp:66-72)
    std::fseek(f.f, 0, SEEK_END);
    const long long size = std::ftell(f.f);
    std::fseek(f.f, 12, SEEK_SET);
    const u64 have = size >= 12 ? static_cast<u64>(size - 12) / 24 : 0;
    require(have >= count, LO_RUNTIME_ERROR,
            p + ": truncated record at byte offset " + std::to_string(12 + 24 * have));
    require(count > 0, LO_INVALID_ARGUMENT, "reorder_cloud: empty cloud");
    double* xyz = dalloc_t<double>(ctx, 3 * count);
    void* stage[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    lo_coded* out = nullptr;
    try {
        stage_begin(ctx, "h2d");
        const u64 chunk = std::min<u64>(kChunkRecords, count);
        for (int k = 0; k < 2; ++k) {
            LO_CUDA(cudaHostAlloc(&stage[k], 24 * chunk, cudaHostAllocDefault));
            LO_CUDA(cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming));
        }
        u64 at = 0;
        for (int k = 0; at < count; k ^= 1) {
            const u64 m = std::min<u64>(chunk, count - at);
            LO_CUDA(cudaEventSynchronize(done[k]));  // the copy that last used this buffer
            require(std::fread(stage[k], 24, m, f.f) == m, LO_RUNTIME_ERROR,
                    p + ": truncated record at byte offset " + std::to_string(12 + 24 * at));
            LO_CUDA(cudaMemcpyAsync(xyz + 3 * at, stage[k], 24 * m, cudaMemcpyHostToDevice, ctx->stream));
            LO_CUDA(cudaEventRecord(done[k], ctx->stream));
            at += m;
        }
        stage_end(ctx);
        try {
            out = reorder_device(ctx, xyz, count, curve, level);
        } catch (const Error& e) {
            // read_binary rejects non-finite records itself (io.cpp:73-76)
            const std::string pre = "non-finite coordinate at point ";
            const std::string msg = e.what();
            if (e.status == LO_INVALID_ARGUMENT && msg.rfind(pre, 0) == 0)
                throw Error(LO_RUNTIME_ERROR,
                            p + ": non-finite coordinate in record " + msg.substr(pre.size()));
            throw;
        }
    } catch (...) {
        sync(ctx);
        for (int k = 0; k < 2; ++k) {
            if (stage[k]) cudaFreeHost(stage[k]);
            if (done[k]) cudaEventDestroy(done[k]);
        }
        dfree(ctx, xyz);
        throw;
    }
    sync(ctx);
    for (int k = 0; k < 2; ++k) {
        cudaFreeHost(stage[k]);
        cudaEventDestroy(done[k]);
    }
    dfree(ctx, xyz);
    return out;
}

}  // namespace lo

using namespace lo;

extern "C" {

int lo_reorder_pcb(lo_context* ctx, const char* path, int curve, int level, lo_coded** out) {
    return api_ctx(ctx, [&] { *out = reorder_pcb(ctx, path, curve, level); });
}

int lo_coded_write_pcb(lo_context* ctx, const lo_coded* coded, const char* path) {
    return api_ctx(ctx, [&] {
        require(coded != nullptr && path != nullptr, LO_INVALID_ARGUMENT, "null cloud or path");
        const std::string p(path);
        std::vector<double> xyz(3 * coded->n);
        require(lo_coded_download(ctx, coded, xyz.data(), nullptr, nullptr) == LO_OK, LO_CUDA_ERROR,
                lo_last_error());
        File f(std::fopen(path, "wb"));
        require(f.f != nullptr, LO_RUNTIME_ERROR, "cannot open '" + p + "' for writing");
        require(std::fwrite("PCB1", 1, 4, f.f) == 4, LO_RUNTIME_ERROR, "write failed for '" + p + "'");
        put_le<u64>(f.f, coded->n);
        require(host_is_little_endian(), LO_RUNTIME_ERROR, "big-endian host");
        require(std::fwrite(xyz.data(), 24, coded->n, f.f) == coded->n, LO_RUNTIME_ERROR,
                "write failed for '" + p + "'");
        require(std::fflush(f.f) == 0, LO_RUNTIME_ERROR, "write failed for '" + p + "'");
    });
}

int lo_octree_from_leaves(lo_context* ctx, const lo_coded* coded, const uint64_t* boundaries_host,
                          const uint32_t* offsets_host, uint64_t count, const double disc_box[6],
                          int level, int curve, uint32_t n_max, lo_octree** out) {
    return api_ctx(ctx, [&] {
        require(boundaries_host && offsets_host && disc_box, LO_INVALID_ARGUMENT, "null leaf array");
        *out = octree_from_leaves(ctx, coded, boundaries_host, offsets_host, count, disc_box, level,
                                  curve, n_max);
    });
}

int lo_octree_save(lo_context* ctx, const lo_octree* tree, const char* path) {
    return api_ctx(ctx, [&] {
        require(tree != nullptr && path != nullptr, LO_INVALID_ARGUMENT, "null tree or path");
        const std::string p(path);
        const u64 count = tree->leaves + 1;
        std::vector<u64> b(count);
        std::vector<u32> o(count);
        LO_CUDA(cudaMemcpyAsync(b.data(), tree->bounds, 8 * count, cudaMemcpyDeviceToHost, ctx->stream));
        LO_CUDA(cudaMemcpyAsync(o.data(), tree->offsets, 4 * count, cudaMemcpyDeviceToHost, ctx->stream));
        sync(ctx);
        File f(std::fopen(path, "wb"));
        require(f.f != nullptr, LO_RUNTIME_ERROR, "cannot open '" + p + "' for writing");
        require(std::fwrite("LOC1", 1, 4, f.f) == 4, LO_RUNTIME_ERROR, "write failed for '" + p + "'");
        put_le<u32>(f.f, static_cast<u32>(tree->level));
        put_le<u32>(f.f, tree->curve == LO_MORTON ? 0u : 1u);
        put_le<u32>(f.f, tree->n_max);
        for (int a = 0; a < 6; ++a) put_le<double>(f.f, tree->disc_box[a]);
        put_le<u64>(f.f, count);
        for (u64 v : b) put_le<u64>(f.f, v);
        for (u32 v : o) put_le<u32>(f.f, v);
        require(std::fflush(f.f) == 0, LO_RUNTIME_ERROR, "write failed for '" + p + "'");
    });
}

int lo_octree_load(lo_context* ctx, const lo_coded* coded, const char* path, lo_octree** out) {
    return api_ctx(ctx, [&] {
        require(path != nullptr, LO_INVALID_ARGUMENT, "null path");
        const std::string p(path);
        File f(std::fopen(path, "rb"));
        require(f.f != nullptr, LO_RUNTIME_ERROR, "cannot open '" + p + "'");
        char magic[4];
        require(std::fread(magic, 1, 4, f.f) == 4 && std::memcmp(magic, "LOC1", 4) == 0,
                LO_RUNTIME_ERROR, "linear octree stream: bad magic");
        u32 level = 0, curve = 0, n_max = 0;
        u64 count = 0;
        double box[6];
        bool ok = get_le(f.f, level) && get_le(f.f, curve) && get_le(f.f, n_max);
        for (int a = 0; a < 6 && ok; ++a) ok = get_le(f.f, box[a]);
        ok = ok && get_le(f.f, count);
        require(ok, LO_RUNTIME_ERROR, "linear octree stream: truncated header");
        // a count the file cannot hold is truncation, before any allocation
        const long long pos = std::ftell(f.f);
        std::fseek(f.f, 0, SEEK_END);
        const long long size = std::ftell(f.f);
        std::fseek(f.f, pos, SEEK_SET);
        require(count <= static_cast<u64>(size - pos) / 12, LO_RUNTIME_ERROR, "linear octree stream: truncated");
        std::vector<u64> b(count);
        std::vector<u32> o(count);
        for (auto& v : b) require(get_le(f.f, v), LO_RUNTIME_ERROR, "linear octree stream: truncated");
        for (auto& v : o) require(get_le(f.f, v), LO_RUNTIME_ERROR, "linear octree stream: truncated");
        *out = octree_from_leaves(ctx, coded, b.data(), o.data(), count, box, static_cast<int>(level),
                                  curve == 0 ? LO_MORTON : LO_HILBERT, n_max);
    });
}

}  // extern "C"
