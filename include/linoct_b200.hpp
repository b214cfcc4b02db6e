// linoct_b200.hpp -- header-only C++ shim with the reference's entry-point shapes
// (proj/include/linoct/{geometry,sfc,reorder,linear_octree,search}.hpp) over the C ABI of
// linoct_b200.h.  Everything runs on the B200; there is no CPU path.  Errors come back as the
// reference's exception types: std::invalid_argument, std::domain_error, std::logic_error,
// std::runtime_error (CUDA / out of memory / no device).
//
//   linoct::b200::PointCloud cloud(points);
//   auto coded = linoct::b200::reorder_cloud(cloud, linoct::b200::Curve::Hilbert);
//   linoct::b200::LinearOctree tree(coded, 32);
//   auto res = linoct::b200::run_radius_batch(tree, coded, RadiusMethod::Lin,
//                                             KernelShape::Sphere, 2.5, BatchOptions{});
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "linoct_b200.h"

namespace linoct::b200 {

inline void check(int status) {
    if (status == LO_OK) return;
    const std::string msg = lo_last_error();
    switch (status) {
        case LO_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case LO_DOMAIN_ERROR: throw std::domain_error(msg);
        case LO_LOGIC_ERROR: throw std::logic_error(msg);
        case LO_RUNTIME_ERROR: throw std::runtime_error(msg);
        default: throw std::runtime_error(msg);
    }
}

struct Point {  // geometry.hpp:14-20
    double x = 0.0, y = 0.0, z = 0.0;
    friend bool operator==(const Point&, const Point&) = default;
};
static_assert(sizeof(Point) == 24, "AoS f64 xyz");

enum class Curve { Morton = LO_MORTON, Hilbert = LO_HILBERT };                    // sfc.hpp:17
enum class KernelShape { Sphere = LO_SPHERE, Circle = LO_CIRCLE, Cube = LO_CUBE, Square = LO_SQUARE };
enum class RadiusMethod { Ptr = LO_METHOD_PTR, Lin = LO_METHOD_LIN, Prune = LO_METHOD_PRUNE,
                          Struct = LO_METHOD_STRUCT };                             // search.hpp:108
enum class BatchMode { Full, RandomSubset };                                       // search.hpp:107
inline constexpr int kMaxLevel = 21;

// One device context per process and device, created on first use (stream = private).
class Context {
  public:
    explicit Context(int device = 0, void* stream = nullptr) {
        check(lo_context_create(device, stream, &ctx_));
    }
    ~Context() { lo_context_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    lo_context* get() const { return ctx_; }
    static Context& default_for(int device = 0) {
        static Context c(device);
        return c;
    }

  private:
    lo_context* ctx_ = nullptr;
};

class PointCloud {  // geometry.hpp:60-99 (validation happens on the device during reorder)
  public:
    PointCloud() = default;
    explicit PointCloud(std::vector<Point> pts) : points_(std::move(pts)) {}
    std::size_t size() const { return points_.size(); }
    bool empty() const { return points_.empty(); }
    const Point& operator[](std::size_t i) const { return points_[i]; }
    const std::vector<Point>& points() const { return points_; }

  private:
    std::vector<Point> points_;
};

// CodedCloud (reorder.hpp:14-20): device resident; host copies are downloaded on demand.
class CodedCloud {
  public:
    CodedCloud(lo_coded* h, Context& ctx) : h_(h, &lo_coded_destroy), ctx_(&ctx) {
        check(lo_coded_info_get(h, &info_));
    }
    lo_coded* handle() const { return h_.get(); }
    Context& context() const { return *ctx_; }
    std::size_t size() const { return info_.n; }
    Curve curve() const { return static_cast<Curve>(info_.curve); }
    const lo_coded_info& info() const { return info_; }
    PointCloud cloud() const {
        std::vector<Point> p(info_.n);
        check(lo_coded_download(ctx_->get(), h_.get(), &p[0].x, nullptr, nullptr));
        return PointCloud(std::move(p));
    }
    std::vector<std::uint64_t> codes() const {
        std::vector<std::uint64_t> c(info_.n);
        check(lo_coded_download(ctx_->get(), h_.get(), nullptr, c.data(), nullptr));
        return c;
    }
    std::vector<std::uint32_t> permutation() const {
        std::vector<std::uint32_t> p(info_.n);
        check(lo_coded_download(ctx_->get(), h_.get(), nullptr, nullptr, p.data()));
        return p;
    }

  private:
    std::shared_ptr<lo_coded> h_;
    Context* ctx_;
    lo_coded_info info_{};
};

// reorder.hpp:23-28
inline std::vector<std::uint64_t> compute_codes(const PointCloud& cloud, Curve curve,
                                                Context& ctx = Context::default_for()) {
    std::vector<std::uint64_t> out(cloud.size());
    check(lo_compute_codes(ctx.get(), cloud.empty() ? nullptr : &cloud[0].x, cloud.size(),
                           static_cast<int>(curve), kMaxLevel, nullptr, out.data()));
    return out;
}

// reorder.hpp:33
inline CodedCloud reorder_cloud(const PointCloud& cloud, Curve curve, int level = kMaxLevel,
                                Context& ctx = Context::default_for()) {
    lo_coded* h = nullptr;
    check(lo_reorder(ctx.get(), cloud.empty() ? nullptr : &cloud[0].x, cloud.size(),
                     static_cast<int>(curve), level, &h));
    return CodedCloud(h, ctx);
}

// reorder_cloud(read_cloud(path), curve, level) for a PCB1 file, streamed to the device
// (io.cpp:53-81); malformed files throw std::runtime_error with the reference's texts.
inline CodedCloud reorder_pcb(const std::string& path, Curve curve, int level = kMaxLevel,
                              Context& ctx = Context::default_for()) {
    lo_coded* h = nullptr;
    check(lo_reorder_pcb(ctx.get(), path.c_str(), static_cast<int>(curve), level, &h));
    return CodedCloud(h, ctx);
}
// write_cloud(coded.cloud, path, BinaryPcb) (io.cpp:94-106)
inline void write_pcb(const CodedCloud& coded, const std::string& path) {
    check(lo_coded_write_pcb(coded.context().get(), coded.handle(), path.c_str()));
}

// reorder.hpp:36
inline std::vector<std::uint32_t> invert_permutation(const std::vector<std::uint32_t>& perm,
                                                     Context& ctx = Context::default_for()) {
    std::vector<std::uint32_t> inv(perm.size());
    check(lo_invert_permutation(ctx.get(), perm.data(), perm.size(), inv.data()));
    return inv;
}

struct LeafArray {  // linear_octree.hpp:20-27
    std::vector<std::uint64_t> boundaries;
    std::vector<std::uint32_t> offsets;
    std::size_t leaf_count() const { return boundaries.size() - 1; }
};

// linear_octree.hpp:33-34 (threads accepted and ignored)
inline LeafArray build_leaves(const std::vector<std::uint64_t>& codes, std::uint32_t n_max,
                              int level = kMaxLevel, int /*threads*/ = 1,
                              Context& ctx = Context::default_for()) {
    std::uint64_t leaves = 0;
    check(lo_build_leaves(ctx.get(), codes.data(), codes.size(), n_max, level, &leaves, nullptr,
                          nullptr, 0));
    LeafArray la{std::vector<std::uint64_t>(leaves + 1), std::vector<std::uint32_t>(leaves + 1)};
    check(lo_build_leaves(ctx.get(), codes.data(), codes.size(), n_max, level, &leaves,
                          la.boundaries.data(), la.offsets.data(), leaves + 1));
    return la;
}

// LinearOctree (linear_octree.hpp:40-118)
class LinearOctree {
  public:
    using NodeRef = std::int32_t;
    using InternalNode = lo_internal_node;

    LinearOctree(const CodedCloud& coded, std::uint32_t n_max = 128, int /*threads*/ = 1)
        : ctx_(&coded.context()) {
        lo_octree* h = nullptr;
        check(lo_octree_build(ctx_->get(), coded.handle(), n_max, &h));
        h_.reset(h, &lo_octree_destroy);
        check(lo_octree_info_get(h, &info_));
    }
    // LinearOctree(LeafArray, Discretizer, Curve, n_max) (linear_octree.cpp:84-105); the leaves
    // must index `coded`'s points, which the device tree searches.
    LinearOctree(const CodedCloud& coded, const LeafArray& leaf_array, const std::array<double, 6>& disc_box,
                 int level, Curve curve, std::uint32_t n_max)
        : ctx_(&coded.context()) {
        if (leaf_array.boundaries.size() != leaf_array.offsets.size())
            throw std::invalid_argument("linear octree: malformed leaf array");
        lo_octree* h = nullptr;
        check(lo_octree_from_leaves(ctx_->get(), coded.handle(), leaf_array.boundaries.data(),
                                    leaf_array.offsets.data(), leaf_array.boundaries.size(), disc_box.data(),
                                    level, static_cast<int>(curve), n_max, &h));
        adopt(h);
    }
    // LinearOctree::serialize / deserialize (linear_octree.cpp:149-190) as LOC1 files.
    void serialize(const std::string& path) const { check(lo_octree_save(ctx_->get(), h_.get(), path.c_str())); }
    static LinearOctree deserialize(const std::string& path, const CodedCloud& coded) {
        lo_octree* h = nullptr;
        check(lo_octree_load(coded.context().get(), coded.handle(), path.c_str(), &h));
        return LinearOctree(h, coded.context());
    }
    lo_octree* handle() const { return h_.get(); }
    static bool is_leaf(NodeRef r) { return r < 0; }
    static std::uint32_t leaf_id(NodeRef r) { return static_cast<std::uint32_t>(~r); }
    static NodeRef leaf_ref(std::uint32_t id) { return ~static_cast<NodeRef>(id); }
    NodeRef root() const { return info_.root; }
    std::size_t leaf_count() const { return info_.leaves; }
    std::size_t internal_count() const { return info_.internal; }
    std::size_t node_count() const { return leaf_count() + internal_count(); }
    std::size_t point_count() const { return info_.points; }
    std::uint32_t n_max() const { return info_.n_max; }
    int level() const { return info_.level; }
    const LeafArray& leaves() const {
        fetch();
        return leaves_;
    }
    const std::vector<InternalNode>& internal_nodes() const {
        fetch();
        return nodes_;
    }
    std::pair<std::uint32_t, std::uint32_t> points_in_node(NodeRef r) const {
        fetch();
        if (is_leaf(r)) return {leaves_.offsets[leaf_id(r)], leaves_.offsets[leaf_id(r) + 1]};
        return {nodes_[r].begin, nodes_[r].end};
    }
    // node_bounds (linear_octree.cpp:139-147): {minx, miny, minz, maxx, maxy, maxz}
    std::array<double, 6> node_bounds(NodeRef r) const {
        std::array<double, 6> b{};
        check(lo_octree_node_bounds(ctx_->get(), h_.get(), &r, 1, b.data()));
        return b;
    }

  private:
    LinearOctree(lo_octree* h, Context& ctx) : ctx_(&ctx) { adopt(h); }
    void adopt(lo_octree* h) {
        h_.reset(h, &lo_octree_destroy);
        check(lo_octree_info_get(h, &info_));
    }
    void fetch() const {
        if (fetched_) return;
        leaves_.boundaries.resize(info_.leaves + 1);
        leaves_.offsets.resize(info_.leaves + 1);
        nodes_.resize(info_.internal);
        check(lo_octree_download(ctx_->get(), h_.get(), leaves_.boundaries.data(),
                                 leaves_.offsets.data(), nodes_.empty() ? nullptr : nodes_.data()));
        fetched_ = true;
    }
    std::shared_ptr<lo_octree> h_;
    Context* ctx_;
    lo_octree_info info_{};
    mutable bool fetched_ = false;
    mutable LeafArray leaves_;
    mutable std::vector<InternalNode> nodes_;
};

struct BatchOptions {  // search.hpp:110-117
    BatchMode mode = BatchMode::Full;
    std::uint32_t subset_size = 5000;
    std::uint64_t seed = 0;
    int threads = 1;
    bool collect_results = false;
    bool fingerprint = true;
};

struct BatchResult {  // search.hpp:121-131 (results as CSR: offsets + indices)
    std::vector<std::uint32_t> centers;
    std::vector<std::uint32_t> counts;
    std::vector<std::uint64_t> fingerprints;
    std::vector<std::uint64_t> offsets;
    std::vector<std::uint32_t> indices;
    std::vector<double> distances;  // kNN only
    double wall_seconds = 0.0;
    double mean_count = 0.0;
    std::vector<std::uint32_t> row(std::size_t i) const {
        return {indices.begin() + offsets[i], indices.begin() + offsets[i + 1]};
    }
};

struct KnnNeighbor {  // search.hpp:80-85
    std::uint32_t index;
    double dist_sq;
    friend bool operator==(const KnnNeighbor&, const KnnNeighbor&) = default;
};

namespace detail {
inline std::vector<std::uint32_t> centres(const CodedCloud& coded, const BatchOptions& o) {
    if (o.mode == BatchMode::Full) return {};
    if (o.subset_size > coded.size()) throw std::invalid_argument("batch: subset size exceeds cloud size");
    std::vector<std::uint32_t> c(o.subset_size);
    check(lo_sample_indices(static_cast<std::uint32_t>(coded.size()), o.subset_size, o.seed, c.data()));
    return c;
}
}  // namespace detail

// search.hpp:135-137
inline BatchResult run_radius_batch(const LinearOctree& tree, const CodedCloud& coded,
                                    RadiusMethod method, KernelShape shape, double radius,
                                    const BatchOptions& options) {
    BatchResult r;
    std::vector<std::uint32_t> c = detail::centres(coded, options);
    lo_csr* h = nullptr;
    check(lo_radius(coded.context().get(), tree.handle(), coded.handle(), static_cast<int>(method),
                    static_cast<int>(shape), radius, c.empty() ? nullptr : c.data(), c.size(),
                    options.fingerprint ? 1 : 0, &h));
    std::unique_ptr<lo_csr, int (*)(lo_csr*)> guard(h, &lo_csr_destroy);
    lo_csr_info info{};
    check(lo_csr_info_get(h, &info));
    r.counts.resize(info.rows);
    if (options.fingerprint) r.fingerprints.resize(info.rows);
    if (options.collect_results) {
        r.offsets.resize(info.rows + 1);
        r.indices.resize(info.total);
    }
    check(lo_csr_download(coded.context().get(), h, r.counts.data(),
                          options.fingerprint ? r.fingerprints.data() : nullptr,
                          options.collect_results ? r.offsets.data() : nullptr,
                          options.collect_results ? r.indices.data() : nullptr));
    if (c.empty()) {
        r.centers.resize(info.rows);
        for (std::uint32_t i = 0; i < info.rows; ++i) r.centers[i] = i;
    } else {
        r.centers = std::move(c);
    }
    r.wall_seconds = info.device_ms * 1e-3;
    r.mean_count = info.mean_count;
    return r;
}

// search.hpp:145-146
inline BatchResult run_knn_batch(const LinearOctree& tree, const CodedCloud& coded, std::uint32_t k,
                                 const BatchOptions& options) {
    BatchResult r;
    std::vector<std::uint32_t> c = detail::centres(coded, options);
    lo_knn_result* h = nullptr;
    check(lo_knn(coded.context().get(), tree.handle(), coded.handle(), k, c.empty() ? nullptr : c.data(),
                 c.size(), options.fingerprint ? 1 : 0, &h));
    std::unique_ptr<lo_knn_result, int (*)(lo_knn_result*)> guard(h, &lo_knn_destroy);
    std::uint64_t rows = 0;
    std::uint32_t keff = 0;
    double ms = 0.0;
    check(lo_knn_info_get(h, &rows, &keff, &ms));
    if (options.fingerprint) r.fingerprints.resize(rows);
    if (options.collect_results) {
        r.indices.resize(rows * keff);
        r.distances.resize(rows * keff);
        r.offsets.resize(rows + 1);
        for (std::uint64_t i = 0; i <= rows; ++i) r.offsets[i] = i * keff;
    }
    check(lo_knn_download(coded.context().get(), h,
                          options.collect_results ? r.indices.data() : nullptr,
                          options.collect_results ? r.distances.data() : nullptr,
                          options.fingerprint ? r.fingerprints.data() : nullptr));
    r.counts.assign(rows, keff);
    if (c.empty()) {
        r.centers.resize(rows);
        for (std::uint32_t i = 0; i < rows; ++i) r.centers[i] = i;
    } else {
        r.centers = std::move(c);
    }
    r.wall_seconds = ms * 1e-3;
    r.mean_count = keff;
    return r;
}

// search.hpp:101-105 at one centre
inline std::vector<KnnNeighbor> knn_lin_oct(const LinearOctree& tree, const CodedCloud& coded,
                                            const Point& center, std::uint32_t k) {
    lo_knn_result* h = nullptr;
    check(lo_knn_points(coded.context().get(), tree.handle(), coded.handle(), k, &center.x, 1, &h));
    std::unique_ptr<lo_knn_result, int (*)(lo_knn_result*)> guard(h, &lo_knn_destroy);
    std::uint64_t rows = 0;
    std::uint32_t keff = 0;
    check(lo_knn_info_get(h, &rows, &keff, nullptr));
    std::vector<std::uint32_t> idx(keff);
    std::vector<double> dist(keff);
    check(lo_knn_download(coded.context().get(), h, idx.data(), dist.data(), nullptr));
    std::vector<KnnNeighbor> out(keff);
    for (std::uint32_t i = 0; i < keff; ++i) out[i] = {idx[i], dist[i]};
    return out;
}

// search.hpp:61-71 at one kernel (Lin and Prune give the same ascending index list)
inline std::vector<std::uint32_t> neighbours_lin(const LinearOctree& tree, const CodedCloud& coded,
                                                 KernelShape shape, const Point& center, double radius) {
    lo_csr* h = nullptr;
    check(lo_radius_points(coded.context().get(), tree.handle(), coded.handle(), static_cast<int>(shape),
                           radius, &center.x, 1, &h));
    std::unique_ptr<lo_csr, int (*)(lo_csr*)> guard(h, &lo_csr_destroy);
    lo_csr_info info{};
    check(lo_csr_info_get(h, &info));
    std::vector<std::uint32_t> idx(info.total);
    check(lo_csr_download(coded.context().get(), h, nullptr, nullptr, nullptr, idx.data()));
    return idx;
}
inline std::vector<std::uint32_t> neighbours_prune(const LinearOctree& tree, const CodedCloud& coded,
                                                   KernelShape shape, const Point& center, double radius) {
    return neighbours_lin(tree, coded, shape, center, radius);
}

// search.hpp:18-56: contained octants as coalesced [begin, end) ranges plus the singles.
struct RangedResult {
    std::vector<std::pair<std::uint32_t, std::uint32_t>> ranges;
    std::vector<std::uint32_t> singles;
    std::size_t count() const {
        std::size_t n = singles.size();
        for (const auto& [b, e] : ranges) n += e - b;
        return n;
    }
    std::vector<std::uint32_t> expand() const {  // ascending two-pointer merge
        std::vector<std::uint32_t> out;
        out.reserve(count());
        std::size_t r = 0, s = 0;
        while (r < ranges.size() || s < singles.size()) {
            if (s == singles.size() || (r < ranges.size() && ranges[r].first < singles[s])) {
                for (std::uint32_t i = ranges[r].first; i < ranges[r].second; ++i) out.push_back(i);
                ++r;
            } else {
                out.push_back(singles[s++]);
            }
        }
        return out;
    }
};

// Ranged rows of a Struct result handle (one RangedResult per row).
inline std::vector<RangedResult> struct_rows(const Context& ctx, const lo_csr* h, std::size_t rows) {
    std::uint64_t tr = 0, ts = 0;
    check(lo_csr_struct_info(h, &tr, &ts));
    std::vector<std::uint64_t> ro(rows + 1), so(rows + 1);
    std::vector<std::uint32_t> rg(2 * tr), sg(ts);
    check(lo_csr_struct_download(ctx.get(), h, ro.data(), rg.data(), so.data(), sg.data()));
    std::vector<RangedResult> out(rows);
    for (std::size_t i = 0; i < rows; ++i) {
        for (std::uint64_t j = ro[i]; j < ro[i + 1]; ++j) out[i].ranges.emplace_back(rg[2 * j], rg[2 * j + 1]);
        out[i].singles.assign(sg.begin() + so[i], sg.begin() + so[i + 1]);
    }
    return out;
}

// search.hpp:75-78
inline RangedResult neighbours_struct(const LinearOctree& tree, const CodedCloud& coded,
                                      KernelShape shape, const Point& center, double radius) {
    lo_csr* h = nullptr;
    check(lo_radius_struct_points(coded.context().get(), tree.handle(), coded.handle(),
                                  static_cast<int>(shape), radius, &center.x, 1, &h));
    std::unique_ptr<lo_csr, int (*)(lo_csr*)> guard(h, &lo_csr_destroy);
    return std::move(struct_rows(coded.context(), h, 1)[0]);
}

// ---- locality (locality.hpp / locality.cpp) -------------------------------------------------
struct LocalityHistogram {  // locality.hpp:18-40
    std::uint32_t k = 0;
    std::uint64_t cloud_size = 0;
    std::uint64_t centres = 0;
    std::vector<std::pair<std::uint32_t, std::uint64_t>> bins;  // (d, count), ascending d
    std::uint64_t total() const {
        std::uint64_t t = 0;
        for (const auto& [d, c] : bins) t += c;
        return t;
    }
    std::uint64_t count_at(std::uint32_t d) const {
        auto it = std::lower_bound(bins.begin(), bins.end(), d,
                                   [](const auto& b, std::uint32_t v) { return b.first < v; });
        return it != bins.end() && it->first == d ? it->second : 0;
    }
    double mean() const {
        const std::uint64_t t = total();
        if (t == 0) return 0.0;
        double s = 0.0;
        for (const auto& [d, c] : bins) s += static_cast<double>(d) * static_cast<double>(c);
        return s / static_cast<double>(t);
    }
    double stddev() const {
        const std::uint64_t t = total();
        if (t == 0) return 0.0;
        const double mu = mean();
        double s = 0.0;
        for (const auto& [d, c] : bins) {
            const double dd = static_cast<double>(d) - mu;
            s += dd * dd * static_cast<double>(c);
        }
        return std::sqrt(s / static_cast<double>(t));
    }
};

namespace detail {
inline LocalityHistogram locality(const LinearOctree& tree, const CodedCloud& coded, std::uint32_t k,
                                  const std::vector<std::uint32_t>& centres,
                                  const std::vector<std::uint32_t>* index_map) {
    const std::uint64_t n = coded.size();
    if (k < 1) throw std::invalid_argument("locality histogram: k must be >= 1");
    if (k > n) throw std::invalid_argument("locality histogram: k exceeds cloud size");
    if (index_map && index_map->size() != n)
        throw std::invalid_argument("locality histogram: index map size mismatch");
    lo_context* ctx = coded.context().get();
    lo_knn_result* h = nullptr;
    check(lo_knn(ctx, tree.handle(), coded.handle(), k, centres.empty() ? nullptr : centres.data(),
                 centres.size(), 0, &h));
    std::unique_ptr<lo_knn_result, int (*)(lo_knn_result*)> guard(h, &lo_knn_destroy);
    const std::uint32_t* c = centres.empty() ? nullptr : centres.data();
    const std::uint32_t* m = index_map ? index_map->data() : nullptr;
    std::uint64_t nb = 0;
    check(lo_locality_histogram(ctx, h, coded.handle(), c, m, &nb, nullptr, nullptr, 0));
    std::vector<std::uint32_t> d(nb);
    std::vector<std::uint64_t> cnt(nb);
    check(lo_locality_histogram(ctx, h, coded.handle(), c, m, &nb, d.data(), cnt.data(), nb));
    LocalityHistogram out;
    out.k = k;
    out.cloud_size = n;
    out.centres = centres.empty() ? n : centres.size();
    out.bins.resize(nb);
    for (std::uint64_t i = 0; i < nb; ++i) out.bins[i] = {d[i], cnt[i]};
    return out;
}
}  // namespace detail

// locality.hpp:49-58 (threads accepted, ignored)
inline LocalityHistogram locality_histogram(const LinearOctree& tree, const CodedCloud& coded,
                                            std::uint32_t k, int /*threads*/ = 1,
                                            const std::vector<std::uint32_t>* index_map = nullptr) {
    return detail::locality(tree, coded, k, {}, index_map);
}
inline LocalityHistogram locality_histogram_approx(const LinearOctree& tree, const CodedCloud& coded,
                                                   std::uint32_t k, std::uint32_t sample_size,
                                                   std::uint64_t seed, int /*threads*/ = 1,
                                                   const std::vector<std::uint32_t>* index_map = nullptr) {
    if (sample_size > coded.size())
        throw std::invalid_argument("locality histogram: sample size exceeds cloud size");
    std::vector<std::uint32_t> c(sample_size);
    check(lo_sample_indices(static_cast<std::uint32_t>(coded.size()), sample_size, seed, c.data()));
    return detail::locality(tree, coded, k, c, index_map);
}
// locality.cpp:112-140
inline double fisher_pearson_skewness(const LocalityHistogram& h) {
    const std::uint64_t t = h.total();
    if (t == 0) return 0.0;
    const double mu = h.mean(), sigma = h.stddev();
    if (sigma == 0.0) return 0.0;
    double s = 0.0;
    for (const auto& [d, c] : h.bins) {
        const double z = (static_cast<double>(d) - mu) / sigma;
        s += z * z * z * static_cast<double>(c);
    }
    return s / static_cast<double>(t);
}
inline std::array<double, 3> histogram_quantiles(const LocalityHistogram& h) {
    const std::uint64_t t = h.total();
    std::array<double, 3> out{0.0, 0.0, 0.0};
    if (t == 0) return out;
    const std::array<double, 3> q{0.25, 0.5, 0.75};
    std::uint64_t cum = 0;
    std::size_t qi = 0;
    for (const auto& [d, c] : h.bins) {
        cum += c;
        while (qi < 3 && static_cast<double>(cum) >= q[qi] * static_cast<double>(t)) out[qi++] = d;
        if (qi == 3) break;
    }
    return out;
}

// ---- memory model (memory_model.hpp:13-58) --------------------------------------------------
struct MemoryReport {
    std::uint64_t bytes_total = 0, node_count = 0, point_count = 0;
    double rho() const { return point_count == 0 ? 0.0 : double(node_count) / double(point_count); }
    double overhead(double point_bytes = 32.0) const { return double(bytes_total) / (point_bytes * double(point_count)); }
};
inline MemoryReport measure_structure(const LinearOctree& tree) {
    MemoryReport r;
    r.node_count = tree.node_count();
    r.point_count = tree.point_count();
    r.bytes_total = (tree.leaf_count() + 1) * (sizeof(std::uint64_t) + sizeof(std::uint32_t)) +
                    tree.internal_count() * sizeof(lo_internal_node);
    return r;
}

}  // namespace linoct::b200
