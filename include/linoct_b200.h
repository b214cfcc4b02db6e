/*
 * linoct_b200.h -- C ABI of the B200-native SFC reorder / linear octree / radius + kNN path.
 *
 * Drop-in boundary for the reference's C++ entry points (paths relative to
 * /root/reference/proj).  Every entry point names the reference interface it replaces.
 * Plain pointers and sizes only; no exceptions cross this boundary.  Host pointers are
 * named `*_host`, device pointers `*_dev`.  Arrays of points are AoS xyz triples of f64
 * (the layout of std::vector<linoct::Point>, geometry.hpp:14-20).
 *
 * Status codes mirror the reference's exception types:
 *   LO_INVALID_ARGUMENT <-> std::invalid_argument, LO_DOMAIN_ERROR <-> std::domain_error,
 *   LO_LOGIC_ERROR <-> std::logic_error.  lo_last_error() returns the message of the last
 *   failure on the calling host thread.
 *
 * Threading (search.hpp:119-120): calls on one lo_context are serialized by the
 * context's lock, so several host threads may share a context; built handles are read-only.
 * lo_context_destroy must not race other calls on the same context.
 */
#ifndef LINOCT_B200_H
#define LINOCT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LO_ABI_VERSION 1

typedef enum {
    LO_OK = 0,
    LO_INVALID_ARGUMENT = 1,
    LO_DOMAIN_ERROR = 2,
    LO_LOGIC_ERROR = 3,
    LO_OUT_OF_MEMORY = 4,
    LO_CUDA_ERROR = 5,
    LO_NO_DEVICE = 6,
    LO_RUNTIME_ERROR = 7, /* std::runtime_error: unreadable / malformed files (io.cpp, linear_octree.cpp:163-189) */
    LO_NCCL_ERROR = 8     /* NCCL missing or a collective failed (multi-GPU entry points) */
} lo_status;

/* enum class Curve {Morton, Hilbert} (sfc.hpp:17) */
enum { LO_MORTON = 0, LO_HILBERT = 1 };
/* enum class KernelShape {Sphere, Circle, Cube, Square} (geometry.hpp:101) */
enum { LO_SPHERE = 0, LO_CIRCLE = 1, LO_CUBE = 2, LO_SQUARE = 3 };
/* enum class RadiusMethod {Ptr, Lin, Prune, Struct} (search.hpp:108) */
enum { LO_METHOD_PTR = 0, LO_METHOD_LIN = 1, LO_METHOD_PRUNE = 2, LO_METHOD_STRUCT = 3 };

typedef struct lo_context lo_context; /* device, stream, memory pool, stage timers */
typedef struct lo_coded lo_coded;     /* CodedCloud (reorder.hpp:14-20), device resident */
typedef struct lo_octree lo_octree;   /* LinearOctree (linear_octree.hpp:40-118) */
typedef struct lo_csr lo_csr;         /* BatchResult of run_radius_batch (search.hpp:121-131) */
typedef struct lo_knn_result lo_knn_result;        /* BatchResult of run_knn_batch + the (index, dist) lists */

/* LinearOctree::InternalNode, byte-identical (linear_octree.hpp:46-53; 56 bytes). */
typedef struct {
    uint64_t prefix;
    int32_t children[8];
    uint32_t begin;
    uint32_t end;
    uint8_t depth;
    uint8_t child_mask;
    uint8_t pad_[6];
} lo_internal_node;

typedef struct {
    uint64_t n;           /* points */
    int32_t curve;        /* LO_MORTON / LO_HILBERT */
    int32_t level;        /* grid level, <= 21 */
    double disc_box[6];   /* Discretizer bbox: cubified cloud bbox (reorder.cpp:71) */
    double cloud_box[6];  /* PointCloud::bbox() of the input (geometry.hpp:74-81) */
    double scale[3];      /* Discretizer scale per axis (sfc.cpp:77-80) */
} lo_coded_info;

typedef struct {
    uint64_t leaves;      /* LeafArray::leaf_count() */
    uint64_t internal;    /* internal_count() */
    int32_t root;         /* root() NodeRef: >= 0 internal, < 0 is ~leaf */
    uint32_t n_max;
    int32_t level;
    int32_t curve;
    uint64_t points;
    uint64_t tnodes;      /* traversal nodes (non-empty nodes), device side only */
} lo_octree_info;

typedef struct {
    uint64_t rows;        /* centres */
    uint64_t total;       /* neighbours over all rows (u64: cfg3 exceeds 2^32) */
    double mean_count;    /* BatchResult::mean_count (mu) */
    double device_ms;     /* device time of the batch (count + scan + fill [+ digests]) */
} lo_csr_info;

/* ---- context ------------------------------------------------------------------------ */
const char* lo_last_error(void);
int lo_abi_version(void);
/* Number of kernels this library has launched in the process (harness evidence). */
uint64_t lo_launch_count(void);
int lo_device_count(int* count);
/* One context = one device + one CUDA stream.  stream = NULL creates a private stream;
 * otherwise work is enqueued on the given cudaStream_t (e.g. torch's current stream). */
int lo_context_create(int device, void* stream, lo_context** out);
int lo_context_destroy(lo_context* ctx);
/* Waits for the context's compute and copy streams (async downloads included). */
int lo_context_synchronize(lo_context* ctx);
void* lo_context_stream(lo_context* ctx);
/* Makes the context stream wait (on the device, no host sync) for the work the library put on
 * its side streams (row digests on the aux stream, async downloads) -- e.g. before recording an
 * end-of-region event on the context stream. */
int lo_context_join(lo_context* ctx);
/* Context options.
 *   LO_OPT_CENTRE_ORDER (default 1): explicit centre lists (RandomSubset, caller order) are
 *     searched along the curve and their rows scattered back; 0 searches them in the caller's
 *     order (the storage-order ablation, cfg4) -- same results, slower on scattered lists.
 *   LO_OPT_RELEASE_SCRATCH (value 1): frees the persistent radius record arena (sized for the
 *     largest batch so far, capped at a quarter of the free memory when it grows) and the cache
 *     of parked result buffers, for callers that share the GPU between batches. */
enum { LO_OPT_CENTRE_ORDER = 1, LO_OPT_RELEASE_SCRATCH = 2 };
int lo_context_set_option(lo_context* ctx, int option, int64_t value);
/* Per-stage device timers (CUDA events on the context stream); off by default. */
int lo_context_set_timing(lo_context* ctx, int enabled);
/* Copies up to cap (name, ms) pairs of the last timed operations; returns count. */
int lo_context_stage_times(lo_context* ctx, char* names, int name_len, double* ms, int cap);
/* Device buffers for harnesses (bench L2 flush, device-resident inputs). */
int lo_device_alloc(lo_context* ctx, uint64_t bytes, void** out_dev);
int lo_device_free(lo_context* ctx, void* dev);
int lo_memcpy_h2d(lo_context* ctx, void* dst_dev, const void* src_host, uint64_t bytes);
/* Staged uploads for pipelined callers: lo_h2d_begin enqueues the copy on the context's upload
 * stream and returns (use pinned host memory); lo_h2d_wait(slot) makes all work enqueued on the
 * context afterwards wait for that copy -- e.g. upload batch i + 1 while batch i computes, then
 * lo_h2d_wait + lo_reorder_device on it.  slot in [0, 4). */
int lo_h2d_begin(lo_context* ctx, void* dst_dev, const void* src_host, uint64_t bytes, int slot);
int lo_h2d_wait(lo_context* ctx, int slot);
/* Result fences for pipelined callers: lo_d2h_fence(slot) marks every lo_csr_download_async
 * enqueued so far; lo_d2h_wait(slot) blocks the host until those copies have
 * landed -- e.g. double-buffered host results: wait on slot s % 2 before reusing its buffers, fence
 * it after the batch's downloads.  slot in [0, 4). */
int lo_d2h_fence(lo_context* ctx, int slot);
int lo_d2h_wait(lo_context* ctx, int slot);
int lo_memcpy_d2h(lo_context* ctx, void* dst_host, const void* src_dev, uint64_t bytes);
int lo_host_alloc_pinned(uint64_t bytes, void** out_host);
int lo_host_free_pinned(void* host);
/* Writes `bytes` of a scratch buffer (L2 flush between timed iterations). */
int lo_flush_l2(lo_context* ctx, void* scratch_dev, uint64_t bytes);

/* ---- sfc (sfc.hpp:56-83, sfc.cpp:8-73) -------------------------------------------- */
/* Per-point codes in cloud order; replaces compute_codes(cloud, curve) (reorder.hpp:28)
 * and, with disc_box != NULL, compute_codes(cloud, curve, disc) (reorder.hpp:23). */
int lo_compute_codes(lo_context* ctx, const double* xyz_host, uint64_t n, int curve, int level,
                     const double* disc_box /* NULL = cubify(bbox) */, uint64_t* codes_host);
/* Bulk codecs on grid cells (morton_/hilbert_encode, sfc_decode). */
int lo_encode_cells(lo_context* ctx, const uint32_t* cells_host, uint64_t n, int curve,
                    int level, uint64_t* codes_host);
int lo_decode_codes(lo_context* ctx, const uint64_t* codes_host, uint64_t n, int curve,
                    int level, uint32_t* cells_host);

/* ---- reorder (reorder.cpp:66-89) ---------------------------------------------------- */
/* reorder_cloud(cloud, curve, level) -> CodedCloud.  Host input (H2D inside). */
int lo_reorder(lo_context* ctx, const double* xyz_host, uint64_t n, int curve, int level,
               lo_coded** out);
/* Same with the cloud already resident in device memory (AoS f64, n*3). */
int lo_reorder_device(lo_context* ctx, const double* xyz_dev, uint64_t n, int curve, int level,
                      lo_coded** out);
int lo_coded_info_get(const lo_coded* coded, lo_coded_info* out);
/* Download the reordered cloud (AoS), sorted codes and permutation[new] = old; any NULL
 * pointer is skipped. */
int lo_coded_download(lo_context* ctx, const lo_coded* coded, double* xyz_host,
                      uint64_t* codes_host, uint32_t* perm_host);
/* Device pointers of the SoA sorted coordinates / codes / permutation (read only). */
int lo_coded_device_ptrs(const lo_coded* coded, const double** x, const double** y,
                         const double** z, const uint64_t** codes, const uint32_t** perm);
int lo_coded_destroy(lo_coded* coded);
/* Multi-GPU replication: an empty CodedCloud with the given header on this context's
 * device, whose buffers (lo_coded_device_ptrs) are then filled by a broadcast. */
int lo_coded_create_empty(lo_context* ctx, const lo_coded_info* info, lo_coded** out);
/* invert_permutation (reorder.hpp:36) */
int lo_invert_permutation(lo_context* ctx, const uint32_t* perm_host, uint64_t n,
                          uint32_t* inv_host);

/* ---- linear octree (linear_octree.cpp:23-147) --------------------------------------- */
/* build_leaves(codes, n_max, level, threads) (linear_octree.hpp:33-34); sorted codes in,
 * LeafArray out.  Size query: boundaries_host == NULL returns *leaves only. */
int lo_build_leaves(lo_context* ctx, const uint64_t* codes_host, uint64_t n, uint32_t n_max,
                    int level, uint64_t* leaves, uint64_t* boundaries_host,
                    uint32_t* offsets_host, uint64_t cap);
/* LinearOctree(coded, n_max, threads) (linear_octree.hpp:55).  `threads` is ignored. */
int lo_octree_build(lo_context* ctx, const lo_coded* coded, uint32_t n_max, lo_octree** out);
int lo_octree_info_get(const lo_octree* tree, lo_octree_info* out);
/* leaves() boundaries[L+1], offsets[L+1]; internal_nodes() [I]; NULL skips. */
int lo_octree_download(lo_context* ctx, const lo_octree* tree, uint64_t* boundaries_host,
                       uint32_t* offsets_host, lo_internal_node* nodes_host);
/* node_bounds(ref) (linear_octree.cpp:139-147) for a batch of NodeRefs: 6 f64 per ref. */
int lo_octree_node_bounds(lo_context* ctx, const lo_octree* tree, const int32_t* refs_host,
                          uint64_t count, double* boxes_host);
int lo_octree_destroy(lo_octree* tree);
/* Device buffers of a tree (boundaries u64[L+1], offsets u32[L+1], nodes[I], traversal
 * table tnodes*64 bytes) and an empty tree of the same shape for replication. */
int lo_octree_device_ptrs(const lo_octree* tree, void** boundaries, void** offsets, void** nodes,
                          void** tnodes);
int lo_octree_create_empty(lo_context* ctx, const lo_coded* coded, const lo_octree_info* info,
                           lo_octree** out);

/* ---- on-disk formats (io.cpp:53-114; linear_octree.cpp:149-190) ---------------------- */
/* reorder_cloud(read_cloud(path), curve, level) for a PCB1 file: the file is streamed through two
 * pinned buffers, disk reads overlapping the H2D copies.  Malformed files -> LO_RUNTIME_ERROR
 * with the reference's messages (bad magic, truncated count/record, non-finite record). */
int lo_reorder_pcb(lo_context* ctx, const char* path, int curve, int level, lo_coded** out);
/* write_cloud(coded.cloud, path, BinaryPcb): the reordered cloud as PCB1. */
int lo_coded_write_pcb(lo_context* ctx, const lo_coded* coded, const char* path);
/* LinearOctree(LeafArray, Discretizer(disc_box, level), curve, n_max) (linear_octree.cpp:84-105):
 * validates the leaf array like the reference (invalid_argument texts), then links the internal
 * nodes on the device.  count = boundaries.size() = offsets.size(); the leaves must index the
 * points of `coded` (offsets.back() == n, same level and curve). */
int lo_octree_from_leaves(lo_context* ctx, const lo_coded* coded, const uint64_t* boundaries_host,
                          const uint32_t* offsets_host, uint64_t count, const double disc_box[6],
                          int level, int curve, uint32_t n_max, lo_octree** out);
/* The internal-node link of LinearOctree(LeafArray, Discretizer, Curve, n_max)
 * (linear_octree.cpp:84-137) without a cloud: validates the leaf array like the reference and
 * links it on the device; *internal and *root are always set, nodes_host (cap entries) is written
 * when it is large enough.  Searching needs lo_octree_from_leaves with the cloud it indexes. */
int lo_link_leaves(lo_context* ctx, const uint64_t* boundaries_host, const uint32_t* offsets_host, uint64_t count,
                   const double disc_box[6], int level, uint64_t* internal, int32_t* root,
                   lo_internal_node* nodes_host, uint64_t cap);
/* Discretizer::octant_bounds (sfc.cpp:110-127): the depth-`depth` octant (hx, hy, hz) of the
 * discretizer box, padded outward by 2 ulps per side; out = {min xyz, max xyz}. */
int lo_octant_bounds(const double disc_box[6], int level, uint32_t hx, uint32_t hy, uint32_t hz, int depth,
                     double out[6]);
/* LinearOctree::serialize / deserialize as LOC1 files. */
int lo_octree_save(lo_context* ctx, const lo_octree* tree, const char* path);
int lo_octree_load(lo_context* ctx, const lo_coded* coded, const char* path, lo_octree** out);

/* ---- radius search (search.cpp:45-156, :261-351) ------------------------------------ */
/* run_radius_batch(tree, coded, method, shape, radius, options).  centres_host == NULL is
 * BatchMode::Full (every point, in sorted order); otherwise `m` cloud indices.  The CSR
 * (u64 row offsets, u32 ascending indices) stays on the device until downloaded. */
int lo_radius(lo_context* ctx, const lo_octree* tree, const lo_coded* coded, int method,
              int shape, double radius, const uint32_t* centres_host, uint64_t m,
              int fingerprint, lo_csr** out);
/* Same with explicit query points (neighbours_lin(tree, coded, SearchKernel) at arbitrary
 * centres, search.hpp:61-64): queries_host is AoS f64, m*3. */
int lo_radius_points(lo_context* ctx, const lo_octree* tree, const lo_coded* coded, int shape,
                     double radius, const double* queries_host, uint64_t m, lo_csr** out);
/* neighbours_struct(tree, coded, SearchKernel) at explicit centres (search.hpp:75-78): a
 * Struct result (see lo_csr_struct_download), with Struct fingerprints. */
int lo_radius_struct_points(lo_context* ctx, const lo_octree* tree, const lo_coded* coded, int shape,
                            double radius, const double* queries_host, uint64_t m, lo_csr** out);
/* Full mode restricted to the contiguous centre range [begin, end) (a shard of the
 * SFC-ordered queries); row r is centre begin + r, indices stay global. */
int lo_radius_range(lo_context* ctx, const lo_octree* tree, const lo_coded* coded, int method,
                    int shape, double radius, uint64_t begin, uint64_t end, int fingerprint,
                    lo_csr** out);
int lo_csr_info_get(const lo_csr* csr, lo_csr_info* out);
/* counts[m], fingerprints[m] (FNV-1a-64, search.cpp:263-271), offsets[m+1], indices[total]. */
int lo_csr_download(lo_context* ctx, const lo_csr* csr, uint32_t* counts_host,
                    uint64_t* fingerprints_host, uint64_t* offsets_host, uint32_t* indices_host);
/* Same, asynchronously: the copies run on the context's copy stream after the result is
 * complete, so the next batch computes while this one's results travel (use pinned host
 * buffers, lo_host_alloc_pinned).  The host buffers are filled once lo_context_synchronize
 * returns; the result may be destroyed before that (its device buffers are released when the
 * copy has finished). */
int lo_csr_download_async(lo_context* ctx, lo_csr* csr, uint32_t* counts_host,
                          uint64_t* fingerprints_host, uint64_t* offsets_host, uint32_t* indices_host);
int lo_csr_device_ptrs(const lo_csr* csr, const uint64_t** offsets, const uint32_t** indices);
/* RadiusMethod::Struct results (neighbours_struct, search.cpp:76-135; RangedResult,
 * search.hpp:18-56): per row the coalesced contained ranges and the singles, each as a CSR
 * (u64 row offsets; ranges as (begin, end) u32 pairs).  Fingerprints of a Struct result hash
 * ranges, a separator, then singles (search.cpp:325-336); counts/offsets/indices above are
 * the expanded rows (RangedResult::expand).  LO_INVALID_ARGUMENT for a Lin/Prune result. */
int lo_csr_struct_info(const lo_csr* csr, uint64_t* total_ranges, uint64_t* total_singles);
int lo_csr_struct_download(lo_context* ctx, const lo_csr* csr, uint64_t* range_offsets_host,
                           uint32_t* ranges_host, uint64_t* single_offsets_host,
                           uint32_t* singles_host);
int lo_csr_destroy(lo_csr* csr);

/* ---- kNN (search.cpp:158-259, :369-388) --------------------------------------------- */
/* run_knn_batch(tree, coded, k, options): per row min(k, N) (index, dist_sq) ascending by
 * (dist_sq, index).  k < 1 -> LO_INVALID_ARGUMENT. */
int lo_knn(lo_context* ctx, const lo_octree* tree, const lo_coded* coded, uint32_t k,
           const uint32_t* centres_host, uint64_t m, int fingerprint, lo_knn_result** out);
/* knn_lin_oct(tree, coded, Point, k) at arbitrary centres (search.hpp:101-105). */
int lo_knn_points(lo_context* ctx, const lo_octree* tree, const lo_coded* coded, uint32_t k,
                  const double* queries_host, uint64_t m, lo_knn_result** out);
/* Full mode over the contiguous centre range [begin, end). */
int lo_knn_range(lo_context* ctx, const lo_octree* tree, const lo_coded* coded, uint32_t k,
                 uint64_t begin, uint64_t end, int fingerprint, lo_knn_result** out);
/* rows, k_eff (= min(k, N)), device ms */
int lo_knn_info_get(const lo_knn_result* res, uint64_t* rows, uint32_t* k_eff, double* device_ms);
/* idx[m*k_eff], dist[m*k_eff], fingerprints[m]; NULL skips. */
int lo_knn_download(lo_context* ctx, const lo_knn_result* res, uint32_t* idx_host, double* dist_host,
                    uint64_t* fingerprints_host);
/* Same, asynchronously on the context's copy stream (pinned host buffers; filled once
 * lo_context_synchronize / a later lo_d2h_wait returns); the result may be destroyed first. */
int lo_knn_download_async(lo_context* ctx, lo_knn_result* res, uint32_t* idx_host, double* dist_host,
                          uint64_t* fingerprints_host);
int lo_knn_destroy(lo_knn_result* res);

/* ---- locality histogram (locality.cpp:41-97), log2 bins ----------------------------- */
/* bins[b]: count of |map(i) - map(j)| over kNN pairs with b = 0 for d = 0 and
 * floor(log2 d) + 1 otherwise (33 bins).  use_perm = 1 maps through the permutation. */
int lo_locality_log2(lo_context* ctx, const lo_knn_result* res, const lo_coded* coded,
                     const uint32_t* centres_host, int use_perm, uint64_t* bins33_host);

/* Exact histogram (LocalityHistogram::bins, locality.cpp:41-97): ascending distinct d with
 * their counts, d = |map(i) - map(j)| over every (centre i, kNN member j) pair of `res`;
 * index_map_host (n entries) or NULL for identity, centres_host as passed to lo_knn (NULL =
 * Full).  *nbins is always set; d_host / count_host are written when nbins <= cap, so call
 * once with cap = 0 to size.  Statistics (mean, stddev, G1, quartiles) are host arithmetic
 * over these bins in the reference's order (linoct_b200.hpp / linoct.py). */
int lo_locality_histogram(lo_context* ctx, const lo_knn_result* res, const lo_coded* coded,
                          const uint32_t* centres_host, const uint32_t* index_map_host,
                          uint64_t* nbins, uint32_t* d_host, uint64_t* count_host, uint64_t cap);

/* ---- multi-GPU (replaces the OpenMP loop over centres, search.cpp:297) ---- */
/* One process per GPU; each process's context gets an NCCL communicator.  The structure is
 * built once (on `root`) and broadcast; every rank searches its contiguous SFC slice of the
 * centres, [n*rank/G, n*(rank+1)/G); each rank's CSR rows are global rows of the batch and are
 * concatenated by offset (row_base = neighbours of the lower ranks).  Results are identical for
 * any G.  NCCL (libnccl.so.2) is loaded on first use; LO_NCCL_ERROR when it is absent. */
typedef struct lo_comm lo_comm;
#define LO_COMM_ID_BYTES 128
/* ncclGetUniqueId on one rank; the caller ships the 128 bytes to the others (any transport). */
int lo_comm_unique_id(void* id_out);
int lo_comm_init(lo_context* ctx, const void* id, int nranks, int rank, lo_comm** out);
int lo_comm_info(const lo_comm* comm, int* rank, int* nranks);
int lo_comm_destroy(lo_comm* comm);
/* The rank's contiguous slice of n centres (host arithmetic). */
int lo_shard_range(uint64_t n, int rank, int nranks, uint64_t* begin, uint64_t* end);
/* Broadcast (CodedCloud, LinearOctree) from `root`: the root passes its handles (outputs set to
 * NULL; it keeps computing while the broadcast runs on the communicator's stream, and destroying
 * its handles waits for it); the others pass NULL and receive new handles on their context (FP32
 * filter copies are rebuilt locally, not sent).  Timed as the stage "broadcast". */
int lo_broadcast_structure(lo_comm* comm, const lo_coded* coded, const lo_octree* tree, int root,
                           lo_coded** coded_out, lo_octree** tree_out);
/* Single-process replication onto another context / device (cudaMemcpyPeerAsync; the same device
 * works too): new handles on `dst`. */
int lo_structure_copy(lo_context* dst, const lo_coded* coded, const lo_octree* tree, lo_coded** coded_out,
                      lo_octree** tree_out);
/* run_radius_batch in Full mode over this rank's slice: *out holds rows [row_begin, row_begin +
 * rows) with local offsets; global offset = local + *row_base; *total = neighbours of all ranks
 * (one NCCL all-gather of u64 totals). */
int lo_radius_sharded(lo_comm* comm, const lo_octree* tree, const lo_coded* coded, int method, int shape,
                      double radius, int fingerprint, lo_csr** out, uint64_t* row_begin, uint64_t* row_base,
                      uint64_t* total);
/* Work-weighted shard bounds (the radius work follows neighbour counts, and cfg3's
 * cluster rows are ~10x the terrain ones).  lo_weighted_bounds is host arithmetic: sample j stands
 * for queries [j*stride, min((j+1)*stride, n)) with cost (sample_counts[j] + base_cost) per query;
 * bounds[0..nranks] (bounds[0] = 0, bounds[nranks] = n, multiples of `stride` in between) split the
 * cumulative cost evenly.  lo_radius_work_bounds measures them with one radius batch over the first
 * 32 centres (one query tile) of every stride block -- 32/stride of the work, deterministic, so
 * every rank computes the same bounds without communication; stride >= 32, a multiple of 32. */
int lo_weighted_bounds(const uint32_t* sample_counts, uint64_t samples, uint32_t stride, uint64_t n,
                       uint32_t base_cost, int nranks, uint64_t* bounds);
int lo_radius_work_bounds(lo_context* ctx, const lo_octree* tree, const lo_coded* coded, int shape,
                          double radius, uint32_t stride, int nranks, uint64_t* bounds);
/* lo_radius_sharded over the caller's bounds[0..nranks] instead of equal slices. */
int lo_radius_sharded_bounds(lo_comm* comm, const lo_octree* tree, const lo_coded* coded, int method, int shape,
                             double radius, int fingerprint, const uint64_t* bounds, lo_csr** out,
                             uint64_t* row_begin, uint64_t* row_base, uint64_t* total);
/* run_knn_batch in Full mode over this rank's slice (fixed-width rows: no exchange). */
int lo_knn_sharded(lo_comm* comm, const lo_octree* tree, const lo_coded* coded, uint32_t k, int fingerprint,
                   lo_knn_result** out, uint64_t* row_begin);

/* ---- synthetic clouds (host; io.cpp:122-130 and SURVEY.md §8d) ---------------------- */
int lo_generate_uniform(uint64_t n, uint64_t seed, double extent, double* xyz_host);
int lo_generate_terrain(uint64_t n, uint64_t seed, double extent_xy, double* xyz_host);
int lo_generate_mixed(uint64_t n, uint64_t seed, double* xyz_host);
/* sample_indices(n, k, seed) (rng.hpp:46-58) */
int lo_sample_indices(uint32_t n, uint32_t k, uint64_t seed, uint32_t* out_host);

#ifdef __cplusplus
}
#endif
#endif /* LINOCT_B200_H */
