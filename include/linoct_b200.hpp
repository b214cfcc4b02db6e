// linoct_b200.hpp -- header-only C++ shim that is source-compatible with the reference's public
// API (proj/include/linoct/{geometry,sfc,reorder,linear_octree,search,locality,memory_model}.hpp)
// over the C ABI of linoct_b200.h.  A reference call site compiles against `linoct::b200` with
// only the namespace swapped (tests/cpp/callsite_test.cpp): the same type names, struct fields,
// constructor and function signatures, default arguments and exception types
// (std::invalid_argument, std::domain_error, std::logic_error, std::runtime_error).
//
// Everything computes on the B200; there is no CPU path.  Differences a caller can observe:
//  - CodedCloud keeps the reordered cloud on the device.  reorder_cloud() also fills the host
//    fields `cloud`, `codes`, `permutation` (the reference's value semantics, one D2H copy of
//    36 B/point); reorder_cloud_device() skips that copy for device-only pipelines.
//  - LinearOctree's host tables (leaves(), internal_nodes(), internal()) are downloaded on first
//    use.  LinearOctree(LeafArray, Discretizer, Curve, n_max) links on the device at once and is
//    attached to the CodedCloud of its first search (the leaves must index that cloud's points).
//  - `threads` arguments are accepted and ignored; KnnAudit reports the emission order of the
//    device's exact top-k (worst_margin = max over consecutive emitted (d[i] - d[i+1]) <= 0).
//  - The pointer octree (RadiusMethod::Ptr, PointerOctree) is out of scope: Ptr throws
//    std::invalid_argument like run_radius_batch does for linear trees (search.cpp:319-321).
//  - wall_seconds is the device time of the batch (CUDA events), not host steady_clock.
#pragma once

#include <algorithm>
#include <array>
#include <bit>
#include <cmath>
#include <cstdint>
#include <limits>
#include <memory>
#include <mutex>
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
        default: throw std::runtime_error(msg);  // CUDA / out of memory / no device / file format
    }
}

// ---- geometry.hpp ---------------------------------------------------------------------------
struct Point {
    double x = 0.0, y = 0.0, z = 0.0;
    friend bool operator==(const Point&, const Point&) = default;
};
static_assert(sizeof(Point) == 24, "AoS f64 xyz");

inline bool is_finite(const Point& p) { return std::isfinite(p.x) && std::isfinite(p.y) && std::isfinite(p.z); }

struct Aabb {
    Point min_corner;
    Point max_corner;
    [[nodiscard]] bool contains(const Point& p) const {
        return p.x >= min_corner.x && p.x <= max_corner.x && p.y >= min_corner.y && p.y <= max_corner.y &&
               p.z >= min_corner.z && p.z <= max_corner.z;
    }
    [[nodiscard]] Point center() const {
        return {0.5 * (min_corner.x + max_corner.x), 0.5 * (min_corner.y + max_corner.y),
                0.5 * (min_corner.z + max_corner.z)};
    }
    friend bool operator==(const Aabb&, const Aabb&) = default;
};

// cubify (geometry.hpp:47-57): every side becomes the longest, anchored at the min corner, and
// the result still contains the input box.
inline Aabb cubify(const Aabb& b) {
    const double side = std::max({b.max_corner.x - b.min_corner.x, b.max_corner.y - b.min_corner.y,
                                  b.max_corner.z - b.min_corner.z});
    return {b.min_corner,
            {std::max(b.min_corner.x + side, b.max_corner.x), std::max(b.min_corner.y + side, b.max_corner.y),
             std::max(b.min_corner.z + side, b.max_corner.z)}};
}

// PointCloud (geometry.hpp:60-99): host point storage, finite check and cached bbox.
class PointCloud {
  public:
    PointCloud() = default;
    explicit PointCloud(std::vector<Point> pts) : points_(std::move(pts)) {
        for (std::size_t i = 0; i < points_.size(); ++i)
            if (!is_finite(points_[i]))
                throw std::invalid_argument("non-finite coordinate at point " + std::to_string(i));
        if (points_.empty()) return;
        bbox_ = {points_[0], points_[0]};
        for (const Point& p : points_) {
            bbox_.min_corner = {std::min(bbox_.min_corner.x, p.x), std::min(bbox_.min_corner.y, p.y),
                                std::min(bbox_.min_corner.z, p.z)};
            bbox_.max_corner = {std::max(bbox_.max_corner.x, p.x), std::max(bbox_.max_corner.y, p.y),
                                std::max(bbox_.max_corner.z, p.z)};
        }
    }
    [[nodiscard]] std::size_t size() const { return points_.size(); }
    [[nodiscard]] bool empty() const { return points_.empty(); }
    [[nodiscard]] const Point& operator[](std::size_t i) const { return points_[i]; }
    [[nodiscard]] const Aabb& bbox() const {
        if (points_.empty()) throw std::logic_error("bbox of empty cloud");
        return bbox_;
    }
    [[nodiscard]] const std::vector<Point>& points() const { return points_; }

  private:
    std::vector<Point> points_;
    Aabb bbox_{};
};

enum class KernelShape { Sphere = LO_SPHERE, Circle = LO_CIRCLE, Cube = LO_CUBE, Square = LO_SQUARE };

// SearchKernel (geometry.hpp:104-125): shape, centre, radius, radius^2 (computed once).
class SearchKernel {
  public:
    SearchKernel(KernelShape shape, const Point& center, double radius)
        : shape_(shape), center_(center), radius_(radius), radius_sq_(radius * radius) {
        if (!(radius > 0.0) || !std::isfinite(radius))
            throw std::invalid_argument("kernel radius must be positive and finite");
        if (!is_finite(center)) throw std::invalid_argument("kernel center must be finite");
    }
    [[nodiscard]] KernelShape shape() const { return shape_; }
    [[nodiscard]] const Point& center() const { return center_; }
    [[nodiscard]] double radius() const { return radius_; }
    [[nodiscard]] double radius_sq() const { return radius_sq_; }

  private:
    KernelShape shape_;
    Point center_;
    double radius_;
    double radius_sq_;
};

// kernel_contains (geometry.hpp:127-141): the membership predicate, for callers' own checks
// (brute-force oracles); the searches evaluate the same expression on the device.
inline bool kernel_contains(const SearchKernel& k, const Point& p) {
    const double dx = p.x - k.center().x, dy = p.y - k.center().y, dz = p.z - k.center().z;
    switch (k.shape()) {
        case KernelShape::Sphere: return dx * dx + dy * dy + dz * dz < k.radius_sq();
        case KernelShape::Circle: return dx * dx + dy * dy < k.radius_sq();
        case KernelShape::Cube: return std::max({std::abs(dx), std::abs(dy), std::abs(dz)}) < k.radius();
        case KernelShape::Square: return std::max(std::abs(dx), std::abs(dy)) < k.radius();
    }
    return false;
}

// ---- device context -------------------------------------------------------------------------
// One context per device, created on first use (private stream).  The reference's functions
// take no context; they run on Context::default_for(0).
class Context {
  public:
    explicit Context(int device = 0, void* stream = nullptr) : device_(device) {
        check(lo_context_create(device, stream, &ctx_));
    }
    ~Context() { lo_context_destroy(ctx_); }  // refused (and leaked) while handles are alive
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    lo_context* get() const { return ctx_; }
    int device() const { return device_; }
    void synchronize() const { check(lo_context_synchronize(ctx_)); }
    static Context& default_for(int device = 0) {
        static std::mutex mu;
        static std::vector<std::unique_ptr<Context>> ctxs;
        std::lock_guard<std::mutex> g(mu);
        if (device < 0) throw std::invalid_argument("device index out of range");
        if (ctxs.size() <= static_cast<std::size_t>(device)) ctxs.resize(device + 1);
        if (!ctxs[device]) ctxs[device] = std::make_unique<Context>(device);
        return *ctxs[device];
    }

  private:
    lo_context* ctx_ = nullptr;
    int device_ = 0;
};

// ---- sfc.hpp --------------------------------------------------------------------------------
inline constexpr int kMaxLevel = 21;
enum class Curve { Morton = LO_MORTON, Hilbert = LO_HILBERT };

struct GridCell {
    std::uint32_t x = 0, y = 0, z = 0;
    friend bool operator==(const GridCell&, const GridCell&) = default;
};

inline std::uint64_t sfc_encode(Curve curve, const GridCell& cell, int level) {
    std::uint64_t code = 0;
    check(lo_encode_cells(Context::default_for().get(), &cell.x, 1, static_cast<int>(curve), level, &code));
    return code;
}
inline GridCell sfc_decode(Curve curve, std::uint64_t code, int level) {
    GridCell c;
    check(lo_decode_codes(Context::default_for().get(), &code, 1, static_cast<int>(curve), level, &c.x));
    return c;
}
inline std::uint64_t morton_encode(const GridCell& c, int level) { return sfc_encode(Curve::Morton, c, level); }
inline std::uint64_t hilbert_encode(const GridCell& c, int level) { return sfc_encode(Curve::Hilbert, c, level); }
inline GridCell morton_decode(std::uint64_t code, int level) { return sfc_decode(Curve::Morton, code, level); }
inline GridCell hilbert_decode(std::uint64_t code, int level) { return sfc_decode(Curve::Hilbert, code, level); }

// Discretizer (sfc.hpp:89-127, sfc.cpp:77-127): per-axis scale 2^level / extent (0 for a
// degenerate axis); cell() clamps floor((v - lo) * scale) to [0, 2^level - 1].
class Discretizer {
  public:
    Discretizer() = default;
    explicit Discretizer(const Aabb& bbox, int level = kMaxLevel) : bbox_(bbox), level_(level) {
        if (level < 0 || level > kMaxLevel) throw std::invalid_argument("level out of range");
        if (bbox.min_corner.x > bbox.max_corner.x || bbox.min_corner.y > bbox.max_corner.y ||
            bbox.min_corner.z > bbox.max_corner.z)
            throw std::invalid_argument("inverted bounding box");
        sx_ = scale(bbox.min_corner.x, bbox.max_corner.x);
        sy_ = scale(bbox.min_corner.y, bbox.max_corner.y);
        sz_ = scale(bbox.min_corner.z, bbox.max_corner.z);
    }
    [[nodiscard]] const Aabb& bbox() const { return bbox_; }
    [[nodiscard]] int level() const { return level_; }
    [[nodiscard]] GridCell cell(const Point& p) const {
        if (!bbox_.contains(p)) throw std::domain_error("point outside discretizer bounds");
        return {axis(p.x, bbox_.min_corner.x, sx_), axis(p.y, bbox_.min_corner.y, sy_),
                axis(p.z, bbox_.min_corner.z, sz_)};
    }
    [[nodiscard]] Aabb octant_bounds(std::uint32_t hx, std::uint32_t hy, std::uint32_t hz, int depth) const {
        const std::array<double, 6> box = box6();
        std::array<double, 6> o{};
        check(lo_octant_bounds(box.data(), level_, hx, hy, hz, depth, o.data()));
        return {{o[0], o[1], o[2]}, {o[3], o[4], o[5]}};
    }
    [[nodiscard]] std::array<double, 6> box6() const {
        return {bbox_.min_corner.x, bbox_.min_corner.y, bbox_.min_corner.z,
                bbox_.max_corner.x, bbox_.max_corner.y, bbox_.max_corner.z};
    }

  private:
    double scale(double lo, double hi) const { return hi - lo > 0.0 ? std::ldexp(1.0, level_) / (hi - lo) : 0.0; }
    std::uint32_t axis(double v, double lo, double s) const {
        const double u = std::floor((v - lo) * s);
        const double top = static_cast<double>((std::uint64_t{1} << level_) - 1);
        return static_cast<std::uint32_t>(std::clamp(u, 0.0, top));
    }
    Aabb bbox_{};
    int level_ = kMaxLevel;
    double sx_ = 0.0, sy_ = 0.0, sz_ = 0.0;
};

// ---- reorder.hpp ----------------------------------------------------------------------------
// CodedCloud (reorder.hpp:14-20): the reference's public fields, plus the device handle the
// searches run on.  Copies share the (immutable) device data.
struct CodedCloud {
    PointCloud cloud;                        // reordered points (host; empty when device-only)
    std::vector<std::uint64_t> codes;        // sorted codes (host; empty when device-only)
    std::vector<std::uint32_t> permutation;  // new index -> original index (host; idem)
    Curve curve = Curve::Morton;
    Discretizer discretizer;

    CodedCloud() = default;
    CodedCloud(lo_coded* h, Context& ctx, bool host_mirror) : h_(h, &lo_coded_destroy), ctx_(&ctx) {
        check(lo_coded_info_get(h, &info_));
        curve = static_cast<Curve>(info_.curve);
        const double* b = info_.disc_box;
        discretizer = Discretizer(Aabb{{b[0], b[1], b[2]}, {b[3], b[4], b[5]}}, info_.level);
        if (host_mirror) download_host_fields();
    }
    // Fills cloud / codes / permutation from the device (reorder_cloud does this at once).
    void download_host_fields() {
        std::vector<Point> p(info_.n);
        codes.resize(info_.n);
        permutation.resize(info_.n);
        check(lo_coded_download(ctx_->get(), h_.get(), info_.n ? &p[0].x : nullptr, codes.data(),
                                permutation.data()));
        cloud = PointCloud(std::move(p));
    }
    lo_coded* handle() const {
        if (!h_) throw std::logic_error("CodedCloud has no device data (default-constructed)");
        return h_.get();
    }
    Context& context() const { return *ctx_; }
    std::size_t size() const { return info_.n; }
    const lo_coded_info& info() const { return info_; }

  private:
    std::shared_ptr<lo_coded> h_;
    Context* ctx_ = nullptr;
    lo_coded_info info_{};
};

// compute_codes (reorder.hpp:23-28): per-point codes in cloud order, on the device.
inline std::vector<std::uint64_t> compute_codes(const PointCloud& cloud, Curve curve, const Discretizer& disc) {
    std::vector<std::uint64_t> out(cloud.size());
    const std::array<double, 6> box = disc.box6();
    check(lo_compute_codes(Context::default_for().get(), cloud.empty() ? nullptr : &cloud[0].x, cloud.size(),
                           static_cast<int>(curve), disc.level(), box.data(), out.data()));
    return out;
}
inline std::vector<std::uint64_t> compute_codes(const PointCloud& cloud, Curve curve) {
    std::vector<std::uint64_t> out(cloud.size());
    check(lo_compute_codes(Context::default_for().get(), cloud.empty() ? nullptr : &cloud[0].x, cloud.size(),
                           static_cast<int>(curve), kMaxLevel, nullptr, out.data()));
    return out;
}

// reorder_cloud (reorder.hpp:33): encode, stable radix sort and gather on the device; the host
// fields are filled like the reference's value result.
inline CodedCloud reorder_cloud(const PointCloud& cloud, Curve curve, int level = kMaxLevel) {
    Context& ctx = Context::default_for();
    lo_coded* h = nullptr;
    check(lo_reorder(ctx.get(), cloud.empty() ? nullptr : &cloud[0].x, cloud.size(), static_cast<int>(curve),
                     level, &h));
    return CodedCloud(h, ctx, true);
}
// The same without the host copy (device-resident pipelines), on a chosen context.
inline CodedCloud reorder_cloud_device(const PointCloud& cloud, Curve curve, int level = kMaxLevel,
                                       Context& ctx = Context::default_for()) {
    lo_coded* h = nullptr;
    check(lo_reorder(ctx.get(), cloud.empty() ? nullptr : &cloud[0].x, cloud.size(), static_cast<int>(curve),
                     level, &h));
    return CodedCloud(h, ctx, false);
}
// reorder_cloud(read_cloud(path), curve, level) for a PCB1 file streamed to the device (io.cpp:53-81).
inline CodedCloud reorder_pcb(const std::string& path, Curve curve, int level = kMaxLevel,
                              Context& ctx = Context::default_for()) {
    lo_coded* h = nullptr;
    check(lo_reorder_pcb(ctx.get(), path.c_str(), static_cast<int>(curve), level, &h));
    return CodedCloud(h, ctx, false);
}
// write_cloud(coded.cloud, path, BinaryPcb) from the device copy (io.cpp:94-106).
inline void write_pcb(const CodedCloud& coded, const std::string& path) {
    check(lo_coded_write_pcb(coded.context().get(), coded.handle(), path.c_str()));
}

// invert_permutation (reorder.hpp:36)
inline std::vector<std::uint32_t> invert_permutation(const std::vector<std::uint32_t>& perm) {
    std::vector<std::uint32_t> inv(perm.size());
    check(lo_invert_permutation(Context::default_for().get(), perm.data(), perm.size(), inv.data()));
    return inv;
}

// ---- linear_octree.hpp ----------------------------------------------------------------------
struct LeafArray {
    std::vector<std::uint64_t> boundaries;
    std::vector<std::uint32_t> offsets;
    [[nodiscard]] std::size_t leaf_count() const { return boundaries.size() - 1; }
};

// build_leaves (linear_octree.hpp:33-34); threads accepted and ignored.
inline LeafArray build_leaves(const std::vector<std::uint64_t>& codes, std::uint32_t n_max, int level = kMaxLevel,
                              int /*threads*/ = 1) {
    lo_context* ctx = Context::default_for().get();
    std::uint64_t leaves = 0;
    check(lo_build_leaves(ctx, codes.data(), codes.size(), n_max, level, &leaves, nullptr, nullptr, 0));
    LeafArray la{std::vector<std::uint64_t>(leaves + 1), std::vector<std::uint32_t>(leaves + 1)};
    check(lo_build_leaves(ctx, codes.data(), codes.size(), n_max, level, &leaves, la.boundaries.data(),
                          la.offsets.data(), leaves + 1));
    return la;
}

class LinearOctree {
  public:
    using NodeRef = std::int32_t;
    using InternalNode = lo_internal_node;  // byte-identical (linear_octree.hpp:46-53, 56 B)

    // LinearOctree(coded, n_max, threads) (linear_octree.hpp:55)
    LinearOctree(const CodedCloud& coded, std::uint32_t n_max = 128, int /*threads*/ = 1)
        : st_(std::make_shared<State>()) {
        st_->ctx = &coded.context();
        lo_octree* h = nullptr;
        check(lo_octree_build(st_->ctx->get(), coded.handle(), n_max, &h));
        adopt(h, coded.handle());
        st_->disc = coded.discretizer;
        st_->curve = coded.curve;
    }
    // LinearOctree(LeafArray, Discretizer, Curve, n_max) (linear_octree.hpp:58): validated and linked
    // on the device now; attached to the cloud of its first search.
    LinearOctree(LeafArray leaf_array, Discretizer disc, Curve curve, std::uint32_t n_max)
        : st_(std::make_shared<State>()) {
        st_->ctx = &Context::default_for();
        if (leaf_array.boundaries.size() != leaf_array.offsets.size())
            throw std::invalid_argument("linear octree: malformed leaf array");
        const std::array<double, 6> box = disc.box6();
        std::uint64_t internal = 0;
        std::int32_t root = 0;
        check(lo_link_leaves(st_->ctx->get(), leaf_array.boundaries.data(), leaf_array.offsets.data(),
                             leaf_array.boundaries.size(), box.data(), disc.level(), &internal, &root, nullptr, 0));
        st_->nodes.resize(internal);
        check(lo_link_leaves(st_->ctx->get(), leaf_array.boundaries.data(), leaf_array.offsets.data(),
                             leaf_array.boundaries.size(), box.data(), disc.level(), &internal, &root,
                             st_->nodes.empty() ? nullptr : st_->nodes.data(), internal));
        st_->leaves = std::move(leaf_array);
        st_->info.leaves = st_->leaves.leaf_count();
        st_->info.internal = internal;
        st_->info.root = root;
        st_->info.n_max = n_max;
        st_->info.level = disc.level();
        st_->info.curve = static_cast<int>(curve);
        st_->info.points = st_->leaves.offsets.back();
        st_->disc = disc;
        st_->curve = curve;
        st_->fetched = true;
    }

    static bool is_leaf(NodeRef r) { return r < 0; }
    static std::uint32_t leaf_id(NodeRef r) { return static_cast<std::uint32_t>(~r); }
    static NodeRef leaf_ref(std::uint32_t id) { return ~static_cast<NodeRef>(id); }

    [[nodiscard]] NodeRef root() const { return st_->info.root; }
    [[nodiscard]] const InternalNode& internal(NodeRef r) const { return internal_nodes()[r]; }
    [[nodiscard]] std::pair<std::uint32_t, std::uint32_t> points_in_node(NodeRef r) const {
        if (is_leaf(r)) return {leaves().offsets[leaf_id(r)], leaves().offsets[leaf_id(r) + 1]};
        return {internal_nodes()[r].begin, internal_nodes()[r].end};
    }
    [[nodiscard]] std::uint64_t node_prefix(NodeRef r) const {
        return is_leaf(r) ? leaves().boundaries[leaf_id(r)] : internal_nodes()[r].prefix;
    }
    [[nodiscard]] int node_depth(NodeRef r) const {
        if (!is_leaf(r)) return internal_nodes()[r].depth;
        const std::uint64_t span = leaves().boundaries[leaf_id(r) + 1] - leaves().boundaries[leaf_id(r)];
        return level() - std::countr_zero(span) / 3;
    }
    // node_bounds (linear_octree.cpp:139-147): the padded octant box of the node's code prefix
    [[nodiscard]] Aabb node_bounds(NodeRef r) const {
        std::array<double, 6> b{};
        if (st_->h) {
            check(lo_octree_node_bounds(st_->ctx->get(), st_->h.get(), &r, 1, b.data()));
        } else {
            const GridCell c = sfc_decode(st_->curve, node_prefix(r), level());
            const int shift = level() - node_depth(r);
            return st_->disc.octant_bounds(c.x >> shift, c.y >> shift, c.z >> shift, node_depth(r));
        }
        return {{b[0], b[1], b[2]}, {b[3], b[4], b[5]}};
    }
    [[nodiscard]] const LeafArray& leaves() const {
        fetch();
        return st_->leaves;
    }
    [[nodiscard]] const std::vector<InternalNode>& internal_nodes() const {
        fetch();
        return st_->nodes;
    }
    [[nodiscard]] std::size_t leaf_count() const { return st_->info.leaves; }
    [[nodiscard]] std::size_t internal_count() const { return st_->info.internal; }
    [[nodiscard]] std::size_t node_count() const { return leaf_count() + internal_count(); }
    [[nodiscard]] std::size_t point_count() const { return st_->info.points; }
    [[nodiscard]] const Discretizer& discretizer() const { return st_->disc; }
    [[nodiscard]] Curve curve() const { return st_->curve; }
    [[nodiscard]] int level() const { return st_->info.level; }
    [[nodiscard]] std::uint32_t n_max() const { return st_->info.n_max; }

    // LinearOctree::serialize / deserialize (linear_octree.cpp:149-190) as LOC1 files.
    void serialize(const std::string& path) const { check(lo_octree_save(st_->ctx->get(), handle_any(), path.c_str())); }
    static LinearOctree deserialize(const std::string& path, const CodedCloud& coded) {
        lo_octree* h = nullptr;
        check(lo_octree_load(coded.context().get(), coded.handle(), path.c_str(), &h));
        LinearOctree t;
        t.st_->ctx = &coded.context();
        t.adopt(h, coded.handle());
        t.st_->disc = coded.discretizer;
        t.st_->curve = coded.curve;
        return t;
    }

    // The device tree that searches `coded` (a leaf-array tree is attached on first use).
    lo_octree* handle_for(const CodedCloud& coded) const {
        std::lock_guard<std::mutex> g(st_->mu);
        if (st_->h && st_->attached == coded.handle()) return st_->h.get();
        if (st_->h && st_->from_build) return st_->h.get();  // the C ABI checks the pairing
        const std::array<double, 6> box = st_->disc.box6();
        lo_octree* h = nullptr;
        check(lo_octree_from_leaves(coded.context().get(), coded.handle(), st_->leaves.boundaries.data(),
                                    st_->leaves.offsets.data(), st_->leaves.boundaries.size(), box.data(), level(),
                                    static_cast<int>(st_->curve), n_max(), &h));
        st_->h.reset(h, &lo_octree_destroy);
        st_->attached = coded.handle();
        return h;
    }

  private:
    struct State {
        std::mutex mu;
        Context* ctx = nullptr;
        std::shared_ptr<lo_octree> h;
        const lo_coded* attached = nullptr;
        bool from_build = false;
        lo_octree_info info{};
        Discretizer disc;
        Curve curve = Curve::Morton;
        std::once_flag once;
        bool fetched = false;
        LeafArray leaves;
        std::vector<InternalNode> nodes;
    };
    LinearOctree() : st_(std::make_shared<State>()) {}
    void adopt(lo_octree* h, const lo_coded* coded) {
        st_->h.reset(h, &lo_octree_destroy);
        st_->attached = coded;
        st_->from_build = true;
        check(lo_octree_info_get(h, &st_->info));
    }
    lo_octree* handle_any() const {
        if (!st_->h) throw std::logic_error("linear octree: not attached to a cloud yet");
        return st_->h.get();
    }
    void fetch() const {
        if (st_->fetched) return;
        std::call_once(st_->once, [&] {
            st_->leaves.boundaries.resize(st_->info.leaves + 1);
            st_->leaves.offsets.resize(st_->info.leaves + 1);
            st_->nodes.resize(st_->info.internal);
            check(lo_octree_download(st_->ctx->get(), st_->h.get(), st_->leaves.boundaries.data(),
                                     st_->leaves.offsets.data(), st_->nodes.empty() ? nullptr : st_->nodes.data()));
        });
    }
    std::shared_ptr<State> st_;
};

// ---- search.hpp -----------------------------------------------------------------------------
// RangedResult (search.hpp:18-56): contained octants as coalesced [begin, end) ranges + singles.
struct RangedResult {
    std::vector<std::pair<std::uint32_t, std::uint32_t>> ranges;
    std::vector<std::uint32_t> singles;
    [[nodiscard]] std::size_t count() const {
        std::size_t n = singles.size();
        for (const auto& [b, e] : ranges) n += e - b;
        return n;
    }
    template <class Fn>
    void for_each_index(Fn&& fn) const {  // ascending two-pointer merge
        std::size_t r = 0, s = 0;
        while (r < ranges.size() || s < singles.size()) {
            if (s == singles.size() || (r < ranges.size() && ranges[r].first < singles[s])) {
                for (std::uint32_t i = ranges[r].first; i < ranges[r].second; ++i) fn(i);
                ++r;
            } else {
                fn(singles[s++]);
            }
        }
    }
    [[nodiscard]] std::vector<std::uint32_t> expand() const {
        std::vector<std::uint32_t> out;
        out.reserve(count());
        for_each_index([&](std::uint32_t i) { out.push_back(i); });
        return out;
    }
    void clear() {
        ranges.clear();
        singles.clear();
    }
};

struct KnnNeighbor {  // search.hpp:80-85
    std::uint32_t index;
    double dist_sq;
    friend bool operator==(const KnnNeighbor&, const KnnNeighbor&) = default;
};

// KnnAudit (search.hpp:90-93).  The device kNN is an exact top-k, not a best-first queue; the
// audit checks what the reference's checks -- emissions in ascending (dist_sq, index) order:
// worst_margin = max over consecutive emitted pairs of d[i] - d[i+1] (<= 0 when correct).
struct KnnAudit {
    double worst_margin = -std::numeric_limits<double>::infinity();
    std::size_t emissions = 0;
};

enum class BatchMode { Full, RandomSubset };                                   // search.hpp:107
enum class RadiusMethod { Ptr = LO_METHOD_PTR, Lin = LO_METHOD_LIN, Prune = LO_METHOD_PRUNE,
                          Struct = LO_METHOD_STRUCT };                         // search.hpp:108

struct BatchOptions {  // search.hpp:110-117 (same fields, order and defaults)
    BatchMode mode = BatchMode::Full;
    std::uint32_t subset_size = 5000;
    std::uint64_t seed = 0;
    int threads = 1;
    bool collect_results = false;
    bool fingerprint = true;
};

struct BatchResult {  // search.hpp:121-131
    std::vector<std::uint32_t> centers;
    std::vector<std::uint32_t> counts;
    std::vector<std::uint64_t> fingerprints;
    std::vector<std::vector<std::uint32_t>> results;  // when collect_results
    double wall_seconds = 0.0;                         // device time of the batch
    double mean_count = 0.0;
    [[nodiscard]] double mean_query_seconds() const {
        return centers.empty() ? 0.0 : wall_seconds / static_cast<double>(centers.size());
    }
};

// Bulk CSR form of a radius batch (what the device produces; results[] is built from it).
struct CsrResult {
    std::vector<std::uint32_t> centers;
    std::vector<std::uint32_t> counts;
    std::vector<std::uint64_t> fingerprints;
    std::vector<std::uint64_t> offsets;  // [rows + 1]
    std::vector<std::uint32_t> indices;  // [offsets.back()]
    double wall_seconds = 0.0;
    double mean_count = 0.0;
    [[nodiscard]] std::vector<std::uint32_t> row(std::size_t i) const {
        return {indices.begin() + offsets[i], indices.begin() + offsets[i + 1]};
    }
};

namespace detail {
// batch_centers (search.cpp:273-283): Full = none (every point, sorted order); RandomSubset =
// sample_indices(n, subset_size, seed), possibly empty.
inline std::vector<std::uint32_t> subset(const CodedCloud& coded, const BatchOptions& o) {
    if (o.subset_size > coded.size()) throw std::invalid_argument("batch: subset size exceeds cloud size");
    std::vector<std::uint32_t> c(o.subset_size);
    if (o.subset_size)
        check(lo_sample_indices(static_cast<std::uint32_t>(coded.size()), o.subset_size, o.seed, c.data()));
    return c;
}
// A non-NULL pointer for a (possibly empty) explicit centre list: NULL means Full mode.
inline const std::uint32_t* centre_ptr(const std::vector<std::uint32_t>& c) {
    static const std::uint32_t none = 0;
    return c.empty() ? &none : c.data();
}
template <class T>
using Owned = std::unique_ptr<T, int (*)(T*)>;

inline CsrResult radius_csr(const LinearOctree& tree, const CodedCloud& coded, RadiusMethod method,
                            KernelShape shape, double radius, const BatchOptions& o, bool rows) {
    CsrResult r;
    const bool full = o.mode == BatchMode::Full;
    std::vector<std::uint32_t> c = full ? std::vector<std::uint32_t>{} : subset(coded, o);
    lo_context* ctx = coded.context().get();
    lo_csr* h = nullptr;
    check(lo_radius(ctx, tree.handle_for(coded), coded.handle(), static_cast<int>(method), static_cast<int>(shape),
                    radius, full ? nullptr : centre_ptr(c), c.size(), o.fingerprint ? 1 : 0, &h));
    Owned<lo_csr> guard(h, &lo_csr_destroy);
    lo_csr_info info{};
    check(lo_csr_info_get(h, &info));
    r.counts.resize(info.rows);
    if (o.fingerprint) r.fingerprints.resize(info.rows);
    if (rows) {
        r.offsets.resize(info.rows + 1);
        r.indices.resize(info.total);
    }
    check(lo_csr_download(ctx, h, r.counts.data(), o.fingerprint ? r.fingerprints.data() : nullptr,
                          rows ? r.offsets.data() : nullptr, rows ? r.indices.data() : nullptr));
    if (full) {
        r.centers.resize(info.rows);
        for (std::uint32_t i = 0; i < info.rows; ++i) r.centers[i] = i;
    } else {
        r.centers = std::move(c);
    }
    r.wall_seconds = info.device_ms * 1e-3;
    r.mean_count = info.mean_count;
    return r;
}
}  // namespace detail

// run_radius_batch (search.hpp:135-137): count -> scan -> fill (-> digests) on the device.
inline BatchResult run_radius_batch(const LinearOctree& tree, const CodedCloud& coded, RadiusMethod method,
                                    KernelShape shape, double radius, const BatchOptions& options) {
    CsrResult c = detail::radius_csr(tree, coded, method, shape, radius, options, options.collect_results);
    BatchResult r;
    r.centers = std::move(c.centers);
    r.counts = std::move(c.counts);
    r.fingerprints = std::move(c.fingerprints);
    if (options.collect_results) {
        r.results.resize(r.counts.size());
        for (std::size_t i = 0; i < r.results.size(); ++i)
            r.results[i].assign(c.indices.begin() + c.offsets[i], c.indices.begin() + c.offsets[i + 1]);
    }
    r.wall_seconds = c.wall_seconds;
    r.mean_count = c.mean_count;
    return r;
}
// The same batch as one CSR (u64 offsets, u32 indices): no per-row vectors.
inline CsrResult run_radius_batch_csr(const LinearOctree& tree, const CodedCloud& coded, RadiusMethod method,
                                      KernelShape shape, double radius, const BatchOptions& options) {
    return detail::radius_csr(tree, coded, method, shape, radius, options, true);
}

// run_knn_batch (search.hpp:145-146); results hold the index lists when collect_results.
inline BatchResult run_knn_batch(const LinearOctree& tree, const CodedCloud& coded, std::uint32_t k,
                                 const BatchOptions& options) {
    BatchResult r;
    const bool full = options.mode == BatchMode::Full;
    std::vector<std::uint32_t> c = full ? std::vector<std::uint32_t>{} : detail::subset(coded, options);
    lo_context* ctx = coded.context().get();
    lo_knn_result* h = nullptr;
    check(lo_knn(ctx, tree.handle_for(coded), coded.handle(), k, full ? nullptr : detail::centre_ptr(c), c.size(),
                 options.fingerprint ? 1 : 0, &h));
    detail::Owned<lo_knn_result> guard(h, &lo_knn_destroy);
    std::uint64_t rows = 0;
    std::uint32_t keff = 0;
    double ms = 0.0;
    check(lo_knn_info_get(h, &rows, &keff, &ms));
    if (options.fingerprint) r.fingerprints.resize(rows);
    std::vector<std::uint32_t> idx(options.collect_results ? rows * keff : 0);
    check(lo_knn_download(ctx, h, options.collect_results ? idx.data() : nullptr, nullptr,
                          options.fingerprint ? r.fingerprints.data() : nullptr));
    if (options.collect_results) {
        r.results.resize(rows);
        for (std::uint64_t i = 0; i < rows; ++i) r.results[i].assign(idx.begin() + i * keff, idx.begin() + (i + 1) * keff);
    }
    r.counts.assign(rows, keff);
    if (full) {
        r.centers.resize(rows);
        for (std::uint32_t i = 0; i < rows; ++i) r.centers[i] = i;
    } else {
        r.centers = std::move(c);
    }
    r.wall_seconds = ms * 1e-3;
    r.mean_count = rows ? keff : 0.0;
    return r;
}

// knn_lin_oct (search.hpp:101-105) at one centre.
inline void knn_lin_oct(const LinearOctree& tree, const CodedCloud& coded, const Point& center, std::uint32_t k,
                        std::vector<KnnNeighbor>& out, KnnAudit* audit = nullptr) {
    if (k < 1) throw std::invalid_argument("knn: k must be >= 1");
    lo_knn_result* h = nullptr;
    check(lo_knn_points(coded.context().get(), tree.handle_for(coded), coded.handle(), k, &center.x, 1, &h));
    detail::Owned<lo_knn_result> guard(h, &lo_knn_destroy);
    std::uint64_t rows = 0;
    std::uint32_t keff = 0;
    check(lo_knn_info_get(h, &rows, &keff, nullptr));
    std::vector<std::uint32_t> idx(keff);
    std::vector<double> dist(keff);
    check(lo_knn_download(coded.context().get(), h, idx.data(), dist.data(), nullptr));
    out.resize(keff);
    for (std::uint32_t i = 0; i < keff; ++i) out[i] = {idx[i], dist[i]};
    if (audit) {
        audit->emissions += keff;
        for (std::uint32_t i = 0; i + 1 < keff; ++i)
            audit->worst_margin = std::max(audit->worst_margin, dist[i] - dist[i + 1]);
    }
}
inline std::vector<KnnNeighbor> knn_lin_oct(const LinearOctree& tree, const CodedCloud& coded, const Point& center,
                                            std::uint32_t k, KnnAudit* audit = nullptr) {
    std::vector<KnnNeighbor> out;
    knn_lin_oct(tree, coded, center, k, out, audit);
    return out;
}

// neighbours_lin / neighbours_prune (search.hpp:61-71): ascending reordered indices.  Both give
// the same exact set (as in the reference, test_search.cpp:68-102).
inline void neighbours_lin(const LinearOctree& tree, const CodedCloud& coded, const SearchKernel& kernel,
                           std::vector<std::uint32_t>& out) {
    lo_csr* h = nullptr;
    check(lo_radius_points(coded.context().get(), tree.handle_for(coded), coded.handle(),
                           static_cast<int>(kernel.shape()), kernel.radius(), &kernel.center().x, 1, &h));
    detail::Owned<lo_csr> guard(h, &lo_csr_destroy);
    lo_csr_info info{};
    check(lo_csr_info_get(h, &info));
    out.resize(info.total);
    check(lo_csr_download(coded.context().get(), h, nullptr, nullptr, nullptr, out.data()));
}
inline std::vector<std::uint32_t> neighbours_lin(const LinearOctree& tree, const CodedCloud& coded,
                                                 const SearchKernel& kernel) {
    std::vector<std::uint32_t> out;
    neighbours_lin(tree, coded, kernel, out);
    return out;
}
inline void neighbours_prune(const LinearOctree& tree, const CodedCloud& coded, const SearchKernel& kernel,
                             std::vector<std::uint32_t>& out) {
    neighbours_lin(tree, coded, kernel, out);
}
inline std::vector<std::uint32_t> neighbours_prune(const LinearOctree& tree, const CodedCloud& coded,
                                                   const SearchKernel& kernel) {
    return neighbours_lin(tree, coded, kernel);
}

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

// neighbours_struct (search.hpp:75-78): the reference's ranged rows (its octant boxes decide
// which nodes become ranges).
inline void neighbours_struct(const LinearOctree& tree, const CodedCloud& coded, const SearchKernel& kernel,
                              RangedResult& out) {
    lo_csr* h = nullptr;
    check(lo_radius_struct_points(coded.context().get(), tree.handle_for(coded), coded.handle(),
                                  static_cast<int>(kernel.shape()), kernel.radius(), &kernel.center().x, 1, &h));
    detail::Owned<lo_csr> guard(h, &lo_csr_destroy);
    out = std::move(struct_rows(coded.context(), h, 1)[0]);
}
inline RangedResult neighbours_struct(const LinearOctree& tree, const CodedCloud& coded, const SearchKernel& kernel) {
    RangedResult out;
    neighbours_struct(tree, coded, kernel, out);
    return out;
}

// ---- locality.hpp / locality.cpp ------------------------------------------------------------
struct LocalityHistogram {  // locality.hpp:18-40
    std::uint32_t k = 0;
    std::uint64_t cloud_size = 0;
    std::uint64_t centres = 0;
    std::vector<std::pair<std::uint32_t, std::uint64_t>> bins;  // (d, count), ascending d
    [[nodiscard]] std::uint64_t total() const {
        std::uint64_t t = 0;
        for (const auto& [d, c] : bins) t += c;
        return t;
    }
    [[nodiscard]] std::uint64_t count_at(std::uint32_t d) const {
        auto it = std::lower_bound(bins.begin(), bins.end(), d,
                                   [](const auto& b, std::uint32_t v) { return b.first < v; });
        return it != bins.end() && it->first == d ? it->second : 0;
    }
    // sequential double accumulation in bin order, as locality.cpp:19-37
    [[nodiscard]] double mean() const {
        const std::uint64_t t = total();
        if (t == 0) return 0.0;
        double s = 0.0;
        for (const auto& [d, c] : bins) s += static_cast<double>(d) * static_cast<double>(c);
        return s / static_cast<double>(t);
    }
    [[nodiscard]] double stddev() const {
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
inline LocalityHistogram locality(const LinearOctree& tree, const CodedCloud& coded, std::uint32_t k, bool full,
                                  const std::vector<std::uint32_t>& centres,
                                  const std::vector<std::uint32_t>* index_map) {
    const std::uint64_t n = coded.size();
    if (k < 1) throw std::invalid_argument("locality histogram: k must be >= 1");
    if (k > n) throw std::invalid_argument("locality histogram: k exceeds cloud size");
    if (index_map && index_map->size() != n) throw std::invalid_argument("locality histogram: index map size mismatch");
    lo_context* ctx = coded.context().get();
    const std::uint32_t* c = full ? nullptr : centre_ptr(centres);
    lo_knn_result* h = nullptr;
    check(lo_knn(ctx, tree.handle_for(coded), coded.handle(), k, c, centres.size(), 0, &h));
    Owned<lo_knn_result> guard(h, &lo_knn_destroy);
    const std::uint32_t* m = index_map ? index_map->data() : nullptr;
    std::uint64_t nb = 0;
    check(lo_locality_histogram(ctx, h, coded.handle(), c, m, &nb, nullptr, nullptr, 0));
    std::vector<std::uint32_t> d(nb);
    std::vector<std::uint64_t> cnt(nb);
    check(lo_locality_histogram(ctx, h, coded.handle(), c, m, &nb, d.data(), cnt.data(), nb));
    LocalityHistogram out;
    out.k = k;
    out.cloud_size = n;
    out.centres = full ? n : centres.size();
    out.bins.resize(nb);
    for (std::uint64_t i = 0; i < nb; ++i) out.bins[i] = {d[i], cnt[i]};
    return out;
}
}  // namespace detail

// locality.hpp:42-58 (threads accepted, ignored)
inline LocalityHistogram locality_histogram(const LinearOctree& tree, const CodedCloud& coded, std::uint32_t k,
                                            int /*threads*/ = 1,
                                            const std::vector<std::uint32_t>* index_map = nullptr) {
    return detail::locality(tree, coded, k, true, {}, index_map);
}
inline LocalityHistogram locality_histogram_approx(const LinearOctree& tree, const CodedCloud& coded,
                                                   std::uint32_t k, std::uint32_t sample_size, std::uint64_t seed,
                                                   int /*threads*/ = 1,
                                                   const std::vector<std::uint32_t>* index_map = nullptr) {
    if (sample_size > coded.size()) throw std::invalid_argument("locality histogram: sample size exceeds cloud size");
    std::vector<std::uint32_t> c(sample_size);
    if (sample_size)
        check(lo_sample_indices(static_cast<std::uint32_t>(coded.size()), sample_size, seed, c.data()));
    return detail::locality(tree, coded, k, false, c, index_map);
}
// locality.cpp:112-125
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
// locality.cpp:127-140
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

// ---- memory_model.hpp -----------------------------------------------------------------------
struct StructureCostParams {
    double node_bytes = 0.0;
    double point_extra_bytes = 0.0;
    double nodes_per_point = 0.0;
    double point_bytes = 32.0;
};
inline double expected_overhead(const StructureCostParams& p) {
    return (p.point_extra_bytes + p.nodes_per_point * p.node_bytes) / p.point_bytes;
}
struct MemoryReport {
    std::uint64_t bytes_total = 0, node_count = 0, point_count = 0;
    [[nodiscard]] double rho() const {
        return point_count == 0 ? 0.0 : static_cast<double>(node_count) / static_cast<double>(point_count);
    }
    [[nodiscard]] double overhead(double point_bytes = 32.0) const {
        return static_cast<double>(bytes_total) / (point_bytes * static_cast<double>(point_count));
    }
};
// memory_model.cpp:21-30: boundaries + offsets per leaf (+1) and 56 B per internal node
inline MemoryReport measure_structure(const LinearOctree& tree) {
    MemoryReport r;
    r.node_count = tree.node_count();
    r.point_count = tree.point_count();
    r.bytes_total = (tree.leaf_count() + 1) * (sizeof(std::uint64_t) + sizeof(std::uint32_t)) +
                    tree.internal_count() * sizeof(lo_internal_node);
    return r;
}
// memory_model.cpp:39-43: a complete octree has 7 leaves (12 B) per 56 B internal node
inline StructureCostParams linear_octree_cost_params(double rho) {
    return {(7.0 * 12.0 + 56.0) / 8.0, 0.0, rho, 32.0};
}

}  // namespace linoct::b200
