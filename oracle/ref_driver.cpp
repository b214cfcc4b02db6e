// ref_driver.cpp -- C entry points over the UNMODIFIED reference library (TEST/BASELINE ONLY).
//
// Compiled by oracle/Makefile together with the reference sources where they lie under
// /root/reference/proj/src (never copied), into oracle/_ref/libref_linoct.so.  Used by
// tests/ to pin the C restatement (oracle/linoct_oracle.c) and to generate golden vectors,
// and by bench.py as the CPU baseline (`cpu_baseline.kind = "reference"`).  Nothing here is
// on the product path.
#include <algorithm>
#include <bit>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <fstream>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include <omp.h>

#include "linoct/geometry.hpp"
#include "linoct/io.hpp"
#include "linoct/linear_octree.hpp"
#include "linoct/locality.hpp"
#include "linoct/reorder.hpp"
#include "linoct/rng.hpp"
#include "linoct/search.hpp"
#include "linoct/sfc.hpp"

using namespace linoct;

namespace {
thread_local std::string g_err;

std::vector<Point> to_points(const double* xyz, std::uint64_t n) {
    std::vector<Point> pts(n);
    for (std::uint64_t i = 0; i < n; ++i) pts[i] = {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
    return pts;
}

struct Pipeline {
    CodedCloud coded;
    LinearOctree* tree = nullptr;
    ~Pipeline() { delete tree; }
};

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
int ref_max_threads() { return omp_get_max_threads(); }

std::uint64_t ref_morton_encode(std::uint32_t x, std::uint32_t y, std::uint32_t z, int level) {
    return morton_encode({x, y, z}, level);
}
std::uint64_t ref_hilbert_encode(std::uint32_t x, std::uint32_t y, std::uint32_t z, int level) {
    return hilbert_encode({x, y, z}, level);
}
void ref_hilbert_decode(std::uint64_t code, int level, std::uint32_t* out) {
    const GridCell c = hilbert_decode(code, level);
    out[0] = c.x, out[1] = c.y, out[2] = c.z;
}

int ref_octant_bounds(const double* box, std::uint32_t hx, std::uint32_t hy, std::uint32_t hz,
                      int depth, int level, double* out) {
    return guarded([&] {
        const Discretizer d(Aabb{{box[0], box[1], box[2]}, {box[3], box[4], box[5]}}, level);
        const Aabb b = d.octant_bounds(hx, hy, hz, depth);
        const double v[6] = {b.min_corner.x, b.min_corner.y, b.min_corner.z,
                             b.max_corner.x, b.max_corner.y, b.max_corner.z};
        std::memcpy(out, v, sizeof v);
    });
}

// Synthetic uniform cloud exactly as the reference generates it (io.cpp:122-130).
void ref_gen_uniform(std::uint64_t n, std::uint64_t seed, double extent, double* xyz) {
    SyntheticSpec spec;
    spec.kind = SyntheticSpec::Kind::Uniform;
    spec.n = n;
    spec.seed = seed;
    spec.extent = extent;
    const PointCloud c = generate_cloud(spec);
    for (std::uint64_t i = 0; i < n; ++i) {
        xyz[3 * i] = c[i].x, xyz[3 * i + 1] = c[i].y, xyz[3 * i + 2] = c[i].z;
    }
}

void ref_sample_indices(std::uint32_t n, std::uint32_t k, std::uint64_t seed, std::uint32_t* out) {
    const auto v = sample_indices(n, k, seed);
    std::copy(v.begin(), v.end(), out);
}

int ref_compute_codes(const double* xyz, std::uint64_t n, int curve, std::uint64_t* codes) {
    return guarded([&] {
        const PointCloud cloud(to_points(xyz, n));
        const auto c = compute_codes(cloud, curve == 0 ? Curve::Morton : Curve::Hilbert);
        std::copy(c.begin(), c.end(), codes);
    });
}

// reorder_cloud + LinearOctree; timings (seconds) out: [0] reorder, [1] build.
int ref_pipeline_create(const double* xyz, std::uint64_t n, int curve, int level,
                        std::uint32_t n_max, int threads, void** out, double* timings) {
    return guarded([&] {
        auto* p = new Pipeline;
        try {
            const PointCloud cloud(to_points(xyz, n));
            auto t0 = std::chrono::steady_clock::now();
            p->coded = reorder_cloud(cloud, curve == 0 ? Curve::Morton : Curve::Hilbert, level);
            auto t1 = std::chrono::steady_clock::now();
            p->tree = new LinearOctree(p->coded, n_max, threads);
            auto t2 = std::chrono::steady_clock::now();
            if (timings) {
                timings[0] = std::chrono::duration<double>(t1 - t0).count();
                timings[1] = std::chrono::duration<double>(t2 - t1).count();
            }
        } catch (...) {
            delete p;
            throw;
        }
        *out = p;
    });
}

void ref_pipeline_destroy(void* h) { delete static_cast<Pipeline*>(h); }

// Re-run the build alone (timed) on an existing pipeline.
double ref_pipeline_rebuild(void* h, std::uint32_t n_max, int threads) {
    auto* p = static_cast<Pipeline*>(h);
    auto t0 = std::chrono::steady_clock::now();
    auto* t = new LinearOctree(p->coded, n_max, threads);
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    delete p->tree;
    p->tree = t;
    return s;
}

// sizes: [0] n, [1] leaves, [2] internal nodes, [3] root (as int64)
void ref_pipeline_sizes(void* h, std::int64_t* sizes) {
    auto* p = static_cast<Pipeline*>(h);
    sizes[0] = static_cast<std::int64_t>(p->coded.cloud.size());
    sizes[1] = static_cast<std::int64_t>(p->tree->leaf_count());
    sizes[2] = static_cast<std::int64_t>(p->tree->internal_count());
    sizes[3] = p->tree->root();
}

void ref_pipeline_disc(void* h, double* box) {
    auto* p = static_cast<Pipeline*>(h);
    const Aabb& b = p->coded.discretizer.bbox();
    const double v[6] = {b.min_corner.x, b.min_corner.y, b.min_corner.z,
                         b.max_corner.x, b.max_corner.y, b.max_corner.z};
    std::memcpy(box, v, sizeof v);
}

void ref_pipeline_coded(void* h, double* xyz, std::uint64_t* codes, std::uint32_t* perm) {
    auto* p = static_cast<Pipeline*>(h);
    const std::size_t n = p->coded.cloud.size();
    for (std::size_t i = 0; i < n; ++i) {
        if (xyz) {
            xyz[3 * i] = p->coded.cloud[i].x;
            xyz[3 * i + 1] = p->coded.cloud[i].y;
            xyz[3 * i + 2] = p->coded.cloud[i].z;
        }
        if (codes) codes[i] = p->coded.codes[i];
        if (perm) perm[i] = p->coded.permutation[i];
    }
}

// nodes: raw InternalNode records (56 B each, linear_octree.hpp:46-53)
void ref_pipeline_tree(void* h, std::uint64_t* boundaries, std::uint32_t* offsets, void* nodes) {
    auto* p = static_cast<Pipeline*>(h);
    const auto& la = p->tree->leaves();
    std::copy(la.boundaries.begin(), la.boundaries.end(), boundaries);
    std::copy(la.offsets.begin(), la.offsets.end(), offsets);
    const auto& in = p->tree->internal_nodes();
    static_assert(sizeof(LinearOctree::InternalNode) == 56);
    if (!in.empty()) std::memcpy(nodes, in.data(), in.size() * sizeof(LinearOctree::InternalNode));
}

int ref_build_leaves(const std::uint64_t* codes, std::uint64_t n, std::uint32_t n_max, int level,
                     std::uint64_t* boundaries, std::uint32_t* offsets, std::uint64_t cap,
                     std::uint64_t* leaves_out) {
    return guarded([&] {
        const std::vector<std::uint64_t> c(codes, codes + n);
        const LeafArray la = build_leaves(c, n_max, level, 1);
        *leaves_out = la.leaf_count();
        if (la.boundaries.size() <= cap) {
            std::copy(la.boundaries.begin(), la.boundaries.end(), boundaries);
            std::copy(la.offsets.begin(), la.offsets.end(), offsets);
        }
    });
}

// Radius batch (search.cpp:316-351).  mode 0 Full, 1 RandomSubset.  method 1 Lin, 2 Prune,
// 3 Struct.  counts/fps sized to #centres; when row_offsets != null the CSR is written too
// (row_offsets[m+1], indices sized by caller from a previous counts call).  Returns wall s.
double ref_radius(void* h, int method, int shape, double radius, int mode, std::uint32_t subset,
                  std::uint64_t seed, int threads, int fingerprint, std::uint32_t* centers,
                  std::uint32_t* counts, std::uint64_t* fps, std::uint64_t* row_offsets,
                  std::uint32_t* indices, double* mean_count) {
    auto* p = static_cast<Pipeline*>(h);
    BatchOptions o;
    o.mode = mode == 0 ? BatchMode::Full : BatchMode::RandomSubset;
    o.subset_size = subset;
    o.seed = seed;
    o.threads = threads;
    o.collect_results = row_offsets != nullptr;
    o.fingerprint = fingerprint != 0;
    BatchResult r;
    const int rc = guarded([&] {
        r = run_radius_batch(*p->tree, p->coded, static_cast<RadiusMethod>(method),
                             static_cast<KernelShape>(shape), radius, o);
    });
    if (rc != 0) return -1.0;
    const std::size_t m = r.centers.size();
    if (centers) std::copy(r.centers.begin(), r.centers.end(), centers);
    if (counts) std::copy(r.counts.begin(), r.counts.end(), counts);
    if (fps && fingerprint) std::copy(r.fingerprints.begin(), r.fingerprints.end(), fps);
    if (row_offsets) {
        std::uint64_t off = 0;
        for (std::size_t i = 0; i < m; ++i) {
            row_offsets[i] = off;
            std::copy(r.results[i].begin(), r.results[i].end(), indices + off);
            off += r.results[i].size();
        }
        row_offsets[m] = off;
    }
    if (mean_count) *mean_count = r.mean_count;
    return r.wall_seconds;
}

// kNN batch (search.cpp:369-388) with full lists gathered by re-running knn_lin_oct when
// idx != null (the batch API only keeps indices).
double ref_knn(void* h, std::uint32_t k, int mode, std::uint32_t subset, std::uint64_t seed,
               int threads, int fingerprint, std::uint32_t* centers, std::uint32_t* counts,
               std::uint64_t* fps, std::uint32_t* idx, double* dist) {
    auto* p = static_cast<Pipeline*>(h);
    BatchOptions o;
    o.mode = mode == 0 ? BatchMode::Full : BatchMode::RandomSubset;
    o.subset_size = subset;
    o.seed = seed;
    o.threads = threads;
    o.collect_results = false;
    o.fingerprint = fingerprint != 0;
    BatchResult r;
    const int rc = guarded([&] { r = run_knn_batch(*p->tree, p->coded, k, o); });
    if (rc != 0) return -1.0;
    const std::size_t m = r.centers.size();
    if (centers) std::copy(r.centers.begin(), r.centers.end(), centers);
    if (counts) std::copy(r.counts.begin(), r.counts.end(), counts);
    if (fps && fingerprint) std::copy(r.fingerprints.begin(), r.fingerprints.end(), fps);
    if (idx) {
        const std::uint32_t kk = static_cast<std::uint32_t>(
            std::min<std::uint64_t>(k, p->coded.cloud.size()));
#pragma omp parallel for schedule(dynamic) num_threads(threads)
        for (std::int64_t i = 0; i < static_cast<std::int64_t>(m); ++i) {
            std::vector<KnnNeighbor> out;
            knn_lin_oct(*p->tree, p->coded, p->coded.cloud[r.centers[i]], k, out);
            for (std::uint32_t j = 0; j < kk; ++j) {
                idx[i * kk + j] = out[j].index;
                if (dist) dist[i * kk + j] = out[j].dist_sq;
            }
        }
    }
    return r.wall_seconds;
}

// knn_lin_oct at an arbitrary centre (search.hpp:101-105).
int ref_knn_point(void* h, const double* c, std::uint32_t k, std::uint32_t* idx, double* dist,
                  std::uint32_t* count) {
    auto* p = static_cast<Pipeline*>(h);
    return guarded([&] {
        std::vector<KnnNeighbor> out;
        knn_lin_oct(*p->tree, p->coded, Point{c[0], c[1], c[2]}, k, out);
        for (std::size_t j = 0; j < out.size(); ++j) {
            idx[j] = out[j].index;
            dist[j] = out[j].dist_sq;
        }
        *count = static_cast<std::uint32_t>(out.size());
    });
}

// neighbours_lin at an arbitrary centre (search.hpp:61-64); returns count, -1 on error.
std::int64_t ref_radius_point(void* h, int shape, const double* c, double r, std::uint32_t* out,
                              std::uint64_t cap) {
    auto* p = static_cast<Pipeline*>(h);
    std::vector<std::uint32_t> v;
    const int rc = guarded([&] {
        v = neighbours_lin(*p->tree, p->coded,
                           SearchKernel(static_cast<KernelShape>(shape), {c[0], c[1], c[2]}, r));
    });
    if (rc != 0) return -1;
    if (v.size() <= cap) std::copy(v.begin(), v.end(), out);
    return static_cast<std::int64_t>(v.size());
}

// neighbours_struct at an arbitrary centre (search.hpp:75-78): ranges as (begin, end) pairs
// and the singles; returns the member count, -1 on error.  Outputs are written only when
// they fit the capacities; *n_ranges / *n_singles always receive the sizes.
std::int64_t ref_radius_struct_point(void* h, int shape, const double* c, double r,
                                     std::uint32_t* ranges, std::uint64_t cap_ranges,
                                     std::uint32_t* singles, std::uint64_t cap_singles,
                                     std::uint64_t* n_ranges, std::uint64_t* n_singles) {
    auto* p = static_cast<Pipeline*>(h);
    RangedResult rr;
    const int rc = guarded([&] {
        rr = neighbours_struct(*p->tree, p->coded,
                               SearchKernel(static_cast<KernelShape>(shape), {c[0], c[1], c[2]}, r));
    });
    if (rc != 0) return -1;
    *n_ranges = rr.ranges.size();
    *n_singles = rr.singles.size();
    if (rr.ranges.size() <= cap_ranges)
        for (std::size_t j = 0; j < rr.ranges.size(); ++j) {
            ranges[2 * j] = rr.ranges[j].first;
            ranges[2 * j + 1] = rr.ranges[j].second;
        }
    if (rr.singles.size() <= cap_singles) std::copy(rr.singles.begin(), rr.singles.end(), singles);
    return static_cast<std::int64_t>(rr.count());
}

// kNN locality histogram (locality.cpp:91-97), flattened to (d, count) pairs.
std::int64_t ref_locality(void* h, std::uint32_t k, int threads, int use_perm_map,
                          std::uint32_t* bins_d, std::uint64_t* bins_c, std::uint64_t cap) {
    auto* p = static_cast<Pipeline*>(h);
    LocalityHistogram hist;
    const int rc = guarded([&] {
        hist = locality_histogram(*p->tree, p->coded, k, threads,
                                  use_perm_map ? &p->coded.permutation : nullptr);
    });
    if (rc != 0) return -1;
    if (hist.bins.size() <= cap) {
        for (std::size_t i = 0; i < hist.bins.size(); ++i) {
            bins_d[i] = hist.bins[i].first;
            bins_c[i] = hist.bins[i].second;
        }
    }
    return static_cast<std::int64_t>(hist.bins.size());
}

// locality_histogram(_approx) + its statistics (locality.cpp:13-140): out = {mean, stddev,
// G1, Q1, Q2, Q3}; sample = 0 -> exact over all centres.  Returns the bin count, -1 on error.
std::int64_t ref_locality_stats(void* h, std::uint32_t k, int threads, int use_perm_map,
                                std::uint32_t sample, std::uint64_t seed, double* out,
                                std::uint32_t* bins_d, std::uint64_t* bins_c, std::uint64_t cap) {
    auto* p = static_cast<Pipeline*>(h);
    LocalityHistogram hist;
    const auto* map = use_perm_map ? &p->coded.permutation : nullptr;
    const int rc = guarded([&] {
        hist = sample ? locality_histogram_approx(*p->tree, p->coded, k, sample, seed, threads, map)
                      : locality_histogram(*p->tree, p->coded, k, threads, map);
    });
    if (rc != 0) return -1;
    const auto q = histogram_quantiles(hist);
    out[0] = hist.mean();
    out[1] = hist.stddev();
    out[2] = fisher_pearson_skewness(hist);
    out[3] = q[0], out[4] = q[1], out[5] = q[2];
    if (hist.bins.size() <= cap)
        for (std::size_t i = 0; i < hist.bins.size(); ++i) {
            bins_d[i] = hist.bins[i].first;
            bins_c[i] = hist.bins[i].second;
        }
    return static_cast<std::int64_t>(hist.bins.size());
}

// ---- on-disk formats (io.cpp, linear_octree.cpp:149-190) ---------------------------------
// read_cloud(path): returns the count (points written when count <= cap), -1 on error.
std::int64_t ref_read_cloud(const char* path, double* xyz, std::uint64_t cap) {
    PointCloud c;
    const int rc = guarded([&] { c = read_cloud(path); });
    if (rc != 0) return -1;
    if (c.size() <= cap)
        for (std::size_t i = 0; i < c.size(); ++i) {
            xyz[3 * i] = c[i].x;
            xyz[3 * i + 1] = c[i].y;
            xyz[3 * i + 2] = c[i].z;
        }
    return static_cast<std::int64_t>(c.size());
}

int ref_write_cloud(const double* xyz, std::uint64_t n, const char* path) {
    return guarded([&] {
        std::vector<Point> pts(n);
        for (std::uint64_t i = 0; i < n; ++i) pts[i] = {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
        write_cloud(PointCloud(std::move(pts)), path);
    });
}

// LinearOctree::serialize of the pipeline's tree.
int ref_pipeline_save_tree(void* h, const char* path) {
    auto* p = static_cast<Pipeline*>(h);
    return guarded([&] {
        std::ofstream os(path, std::ios::binary | std::ios::trunc);
        p->tree->serialize(os);
        if (!os) throw std::runtime_error("write failed");
    });
}

// LinearOctree::deserialize(path) or LinearOctree(LeafArray, Discretizer, curve, n_max) when
// path is null: leaves / internal nodes / root of the linked tree (sizes always reported;
// arrays written when they fit).
int ref_link_tree(const char* path, const std::uint64_t* b_in, const std::uint32_t* o_in,
                  std::uint64_t count_in, const double* box, int level, int curve, std::uint32_t n_max,
                  std::uint64_t* b_out, std::uint32_t* o_out, std::uint64_t cap, void* nodes,
                  std::uint64_t node_cap, std::uint64_t* leaves, std::uint64_t* internal,
                  std::int32_t* root) {
    return guarded([&] {
        std::unique_ptr<LinearOctree> t;
        if (path) {
            std::ifstream is(path, std::ios::binary);
            if (!is) throw std::runtime_error("cannot open");
            t = std::make_unique<LinearOctree>(LinearOctree::deserialize(is));
        } else {
            LeafArray la;
            la.boundaries.assign(b_in, b_in + count_in);
            la.offsets.assign(o_in, o_in + count_in);
            const Discretizer d(Aabb{{box[0], box[1], box[2]}, {box[3], box[4], box[5]}}, level);
            t = std::make_unique<LinearOctree>(std::move(la), d, curve == 0 ? Curve::Morton : Curve::Hilbert,
                                               n_max);
        }
        const auto& la = t->leaves();
        *leaves = la.leaf_count();
        const auto& in = t->internal_nodes();
        *internal = in.size();
        *root = t->root();
        if (la.boundaries.size() <= cap) {
            std::copy(la.boundaries.begin(), la.boundaries.end(), b_out);
            std::copy(la.offsets.begin(), la.offsets.end(), o_out);
        }
        if (in.size() <= node_cap && !in.empty())
            std::memcpy(nodes, in.data(), in.size() * sizeof(LinearOctree::InternalNode));
    });
}

}  // extern "C"

extern "C" {

// The reference's own per-centre search (neighbours_lin / neighbours_prune,
// search.hpp:61-71) over the contiguous SFC-ordered centre range [begin, end), with the
// batch loop's dynamic OpenMP schedule and FNV digests (search.cpp:287-312, :345-347).
// This is run_batch_loop restricted to a slice, used for bounded CPU-baseline samples.
// Returns wall seconds of the loop (steady_clock, as run_batch_loop measures).
double ref_radius_range(void* h, int method, int shape, double radius, std::uint64_t begin,
                        std::uint64_t end, int threads, std::uint32_t* counts, std::uint64_t* fps) {
    auto* p = static_cast<Pipeline*>(h);
    const std::int64_t m = static_cast<std::int64_t>(end - begin);
    const auto t0 = std::chrono::steady_clock::now();
#pragma omp parallel for schedule(dynamic) num_threads(threads)
    for (std::int64_t i = 0; i < m; ++i) {
        thread_local std::vector<std::uint32_t> idx;
        const SearchKernel kernel(static_cast<KernelShape>(shape),
                                  p->coded.cloud[begin + static_cast<std::uint64_t>(i)], radius);
        if (method == 2) neighbours_prune(*p->tree, p->coded, kernel, idx);
        else neighbours_lin(*p->tree, p->coded, kernel, idx);
        std::uint64_t hsh = 0xcbf29ce484222325ULL;
        for (std::uint32_t v : idx) {
            for (int b = 0; b < 8; ++b) {
                hsh ^= (static_cast<std::uint64_t>(v) >> (8 * b)) & 0xff;
                hsh *= 0x100000001b3ULL;
            }
        }
        if (counts) counts[i] = static_cast<std::uint32_t>(idx.size());
        if (fps) fps[i] = hsh;
    }
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// run_batch_loop (search.cpp:287-312) over an explicit list of centre indices instead of
// batch_centers(): the query of run_radius_batch (search.cpp:322-350, Lin/Prune, FNV digests
// on) for every listed centre, dynamic OpenMP schedule, counts/digests in list order.  The
// bench's reference arm passes many contiguous SFC slices spread over the whole cloud, so a
// bounded sample sees every part of the cloud (clusters, terrain, noise) in proportion.
// Returns the loop's wall seconds (steady_clock, as run_batch_loop measures).
double ref_radius_centres(void* h, int method, int shape, double radius, const std::uint32_t* centres,
                          std::uint64_t m, int threads, std::uint32_t* counts, std::uint64_t* fps) {
    auto* p = static_cast<Pipeline*>(h);
    const auto t0 = std::chrono::steady_clock::now();
#pragma omp parallel for schedule(dynamic) num_threads(threads)
    for (std::int64_t i = 0; i < static_cast<std::int64_t>(m); ++i) {
        thread_local std::vector<std::uint32_t> idx;
        const SearchKernel kernel(static_cast<KernelShape>(shape), p->coded.cloud[centres[i]], radius);
        if (method == 2) neighbours_prune(*p->tree, p->coded, kernel, idx);
        else neighbours_lin(*p->tree, p->coded, kernel, idx);
        std::uint64_t hsh = 0xcbf29ce484222325ULL;
        for (std::uint32_t v : idx) {
            for (int b = 0; b < 8; ++b) {
                hsh ^= (static_cast<std::uint64_t>(v) >> (8 * b)) & 0xff;
                hsh *= 0x100000001b3ULL;
            }
        }
        if (counts) counts[i] = static_cast<std::uint32_t>(idx.size());
        if (fps) fps[i] = hsh;
    }
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// run_knn_batch's query (search.cpp:369-388) over an explicit centre list, digests on.
double ref_knn_centres(void* h, std::uint32_t k, const std::uint32_t* centres, std::uint64_t m,
                       int threads, std::uint64_t* fps) {
    auto* p = static_cast<Pipeline*>(h);
    const auto t0 = std::chrono::steady_clock::now();
#pragma omp parallel for schedule(dynamic) num_threads(threads)
    for (std::int64_t i = 0; i < static_cast<std::int64_t>(m); ++i) {
        thread_local std::vector<KnnNeighbor> found;
        knn_lin_oct(*p->tree, p->coded, p->coded.cloud[centres[i]], k, found);
        std::uint64_t hsh = 0xcbf29ce484222325ULL;
        for (const KnnNeighbor& nb : found) {
            const std::uint64_t vals[2] = {nb.index, std::bit_cast<std::uint64_t>(nb.dist_sq)};
            for (std::uint64_t v : vals)
                for (int b = 0; b < 8; ++b) {
                    hsh ^= (v >> (8 * b)) & 0xff;
                    hsh *= 0x100000001b3ULL;
                }
        }
        if (fps) fps[i] = hsh;
    }
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// knn_lin_oct over [begin, end) (search.cpp:369-388 restricted to a slice).
double ref_knn_range(void* h, std::uint32_t k, std::uint64_t begin, std::uint64_t end, int threads,
                     std::uint64_t* fps) {
    auto* p = static_cast<Pipeline*>(h);
    const std::int64_t m = static_cast<std::int64_t>(end - begin);
    const auto t0 = std::chrono::steady_clock::now();
#pragma omp parallel for schedule(dynamic) num_threads(threads)
    for (std::int64_t i = 0; i < m; ++i) {
        thread_local std::vector<KnnNeighbor> found;
        knn_lin_oct(*p->tree, p->coded, p->coded.cloud[begin + static_cast<std::uint64_t>(i)], k, found);
        std::uint64_t hsh = 0xcbf29ce484222325ULL;
        for (const KnnNeighbor& nb : found) {
            const std::uint64_t vals[2] = {nb.index, std::bit_cast<std::uint64_t>(nb.dist_sq)};
            for (std::uint64_t v : vals)
                for (int b = 0; b < 8; ++b) {
                    hsh ^= (v >> (8 * b)) & 0xff;
                    hsh *= 0x100000001b3ULL;
                }
        }
        if (fps) fps[i] = hsh;
    }
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // extern "C"
