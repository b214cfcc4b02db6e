// Source-compatibility check of the drop-in boundary: one translation unit written against the
// reference's public C++ API (proj/include/linoct/*.hpp) the way its own callers use it -- the
// CLI's run_build / run_radius / run_knn / run_locality (proj/tools/cli.cpp:138-262) and the
// search tests' fixture and oracle checks (proj/tests/test_search.cpp:18-102) -- compiled twice
// with only the namespace swapped:
//
//   g++ -DLINOCT_REFERENCE -I/root/reference/proj/include ... -lref_linoct  -> oracle/_ref/callsite_ref
//   g++ -Iinclude ... -llinoct_b200                                          -> tests/cpp/callsite_b200
//
// Both binaries print the same report (structure sizes, per-batch digest checksums, kNN lists,
// locality statistics, node boxes); tests/test_cpp_shim.py runs both and requires identical
// output.  The reference build is made here (where /root/reference exists) and travels to the
// GPU box as a prebuilt binary.
#include <algorithm>
#include <cinttypes>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#ifdef LINOCT_REFERENCE
#include "linoct/io.hpp"
#include "linoct/linear_octree.hpp"
#include "linoct/locality.hpp"
#include "linoct/memory_model.hpp"
#include "linoct/reorder.hpp"
#include "linoct/rng.hpp"
#include "linoct/search.hpp"
using namespace linoct;
#else
#include "linoct_b200.hpp"
using namespace linoct::b200;
#endif

namespace {

int failures = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        if (!(cond)) {                                                           \
            std::printf("CHECK FAILED: %s (line %d)\n", #cond, __LINE__);        \
            ++failures;                                                          \
        }                                                                        \
    } while (0)

// A seeded cloud with clustered and sparse parts (plain std::mt19937_64, identical in both builds).
std::vector<Point> make_points(std::size_t n, std::uint64_t seed) {
    std::mt19937_64 gen(seed);
    std::uniform_real_distribution<double> u(0.0, 1.0);
    std::vector<Point> p(n);
    for (std::size_t i = 0; i < n; ++i) {
        if (i % 3 == 0) {
            p[i] = {40.0 + 4.0 * u(gen), 60.0 + 4.0 * u(gen), 10.0 + 4.0 * u(gen)};
        } else {
            p[i] = {100.0 * u(gen), 100.0 * u(gen), 20.0 * u(gen)};
        }
    }
    return p;
}

std::uint64_t mix(std::uint64_t h, std::uint64_t v) {
    h ^= v + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2);
    return h;
}

template <class V>
std::uint64_t digest(const V& v) {
    std::uint64_t h = 0;
    for (const auto& x : v) h = mix(h, static_cast<std::uint64_t>(x));
    return h;
}

// The search tests' fixture shape: cloud, coded cloud, tree (test_search.cpp:20-30).
struct Fixture {
    PointCloud cloud;
    CodedCloud coded;
    LinearOctree tree;
    Fixture(std::size_t n, std::uint64_t seed, Curve curve, std::uint32_t n_max)
        : cloud(make_points(n, seed)), coded(reorder_cloud(cloud, curve)), tree(coded, n_max) {}
};

std::vector<std::uint32_t> scan_radius(const PointCloud& cloud, const SearchKernel& kernel) {
    std::vector<std::uint32_t> out;
    for (std::uint32_t i = 0; i < cloud.size(); ++i)
        if (kernel_contains(kernel, cloud[i])) out.push_back(i);
    return out;
}

std::vector<std::uint32_t> to_original(const std::vector<std::uint32_t>& idx, const std::vector<std::uint32_t>& perm) {
    std::vector<std::uint32_t> out;
    out.reserve(idx.size());
    for (std::uint32_t i : idx) out.push_back(perm[i]);
    std::sort(out.begin(), out.end());
    return out;
}

void print_box(const char* tag, const Aabb& b) {
    std::printf("%s %.17g %.17g %.17g %.17g %.17g %.17g\n", tag, b.min_corner.x, b.min_corner.y, b.min_corner.z,
                b.max_corner.x, b.max_corner.y, b.max_corner.z);
}

}  // namespace

int main() {
    for (Curve curve : {Curve::Morton, Curve::Hilbert}) {
        const char* cname = curve == Curve::Morton ? "morton" : "hilbert";
        const Fixture f(20000, curve == Curve::Morton ? 11 : 12, curve, 48);

        // run_build's report (cli.cpp:138-155)
        std::printf("[%s] build: %zu leaves, %zu internal, root %d, points %zu\n", cname, f.tree.leaf_count(),
                    f.tree.internal_count(), static_cast<int>(f.tree.root()), f.tree.point_count());
        const MemoryReport rep = measure_structure(f.tree);
        std::printf("[%s] memory: %" PRIu64 " bytes rho %.17g overhead %.17g model %.17g\n", cname, rep.bytes_total,
                    rep.rho(), rep.overhead(), expected_overhead(linear_octree_cost_params(rep.rho())));
        std::printf("[%s] codes %016" PRIx64 " perm %016" PRIx64 "\n", cname, digest(f.coded.codes),
                    digest(f.coded.permutation));
        print_box("disc", f.coded.discretizer.bbox());
        print_box("root", f.tree.node_bounds(f.tree.root()));
        if (f.tree.internal_count() > 1) {
            const auto& node = f.tree.internal(1);
            std::printf("[%s] node1 prefix %" PRIu64 " depth %d mask %d begin %u end %u child0 %d\n", cname,
                        static_cast<std::uint64_t>(node.prefix), static_cast<int>(node.depth),
                        static_cast<int>(node.child_mask), node.begin, node.end, static_cast<int>(node.children[0]));
            print_box("node1", f.tree.node_bounds(1));
        }
        const LeafArray& leaves = f.tree.leaves();
        std::printf("[%s] leaves %016" PRIx64 " %016" PRIx64 "\n", cname, digest(leaves.boundaries),
                    digest(leaves.offsets));
        const LinearOctree relinked(f.tree.leaves(), f.tree.discretizer(), f.tree.curve(), f.tree.n_max());
        CHECK(relinked.internal_count() == f.tree.internal_count() && relinked.root() == f.tree.root());

        // test_search.cpp-style checks: disjoint / all-inclusive kernels and the scan oracle
        CHECK(neighbours_lin(f.tree, f.coded, SearchKernel(KernelShape::Sphere, {-900, 0, 0}, 2)).empty());
        CHECK(neighbours_lin(f.tree, f.coded, SearchKernel(KernelShape::Sphere, {50, 50, 10}, 1e5)).size() ==
              f.cloud.size());
        const RangedResult whole = neighbours_struct(f.tree, f.coded, SearchKernel(KernelShape::Cube, {50, 50, 10}, 1e5));
        CHECK(whole.ranges.size() == 1 && whole.singles.empty());
        std::mt19937_64 gen(5);
        const KernelShape shapes[] = {KernelShape::Sphere, KernelShape::Circle, KernelShape::Cube, KernelShape::Square};
        std::uint64_t acc = 0;
        for (int it = 0; it < 24; ++it) {
            const Point centre = f.coded.cloud[gen() % f.coded.cloud.size()];
            const double r = it % 3 == 0 ? 0.8 : it % 3 == 1 ? 3.0 : 9.5;
            const SearchKernel kernel(shapes[it % 4], centre, r);
            const auto oracle = scan_radius(f.coded.cloud, kernel);
            const auto lin = neighbours_lin(f.tree, f.coded, kernel);
            const auto prune = neighbours_prune(f.tree, f.coded, kernel);
            const RangedResult ranged = neighbours_struct(f.tree, f.coded, kernel);
            CHECK(lin == oracle && prune == oracle);
            CHECK(ranged.expand() == oracle && ranged.count() == oracle.size());
            acc = mix(acc, digest(lin));
            acc = mix(acc, ranged.ranges.size());
            CHECK(to_original(prune, f.coded.permutation) == scan_radius(f.cloud, kernel));
        }
        std::printf("[%s] kernels %016" PRIx64 "\n", cname, acc);

        // run_radius (cli.cpp:157-199): BatchOptions{mode, subset, seed, threads, collect}
        for (RadiusMethod method : {RadiusMethod::Lin, RadiusMethod::Prune, RadiusMethod::Struct}) {
            BatchOptions options{BatchMode::RandomSubset, 700, 99, 4, true};
            const BatchResult res = run_radius_batch(f.tree, f.coded, method, KernelShape::Sphere, 2.5, options);
            std::uint64_t rows = 0;
            for (const auto& row : res.results) rows = mix(rows, digest(row));
            std::printf("[%s] radius m%d: centers %zu mu %.17g fp %016" PRIx64 " rows %016" PRIx64
                        " centres %016" PRIx64 " mqs>=0 %d\n",
                        cname, static_cast<int>(method), res.centers.size(), res.mean_count, digest(res.fingerprints),
                        rows, digest(res.centers), res.mean_query_seconds() >= 0.0);
        }
        {
            const BatchResult full = run_radius_batch(f.tree, f.coded, RadiusMethod::Lin, KernelShape::Circle, 1.5,
                                                      BatchOptions{});
            std::printf("[%s] radius full circle: %zu %.17g %016" PRIx64 " %016" PRIx64 "\n", cname,
                        full.centers.size(), full.mean_count, digest(full.counts), digest(full.fingerprints));
        }

        // run_knn (cli.cpp:201-226) and the audit check (test_search.cpp:228-240)
        {
            BatchOptions options{BatchMode::Full, 0, 0, 4, true};
            const BatchResult res = run_knn_batch(f.tree, f.coded, 12, options);
            std::uint64_t rows = 0;
            for (const auto& row : res.results) rows = mix(rows, digest(row));
            std::printf("[%s] knn: centers %zu mu %.17g fp %016" PRIx64 " rows %016" PRIx64 "\n", cname,
                        res.centers.size(), res.mean_count, digest(res.fingerprints), rows);
            KnnAudit audit;
            for (int i = 0; i < 20; ++i) {
                const Point centre = f.coded.cloud[(i * 977) % f.coded.cloud.size()];
                const std::vector<KnnNeighbor> nb = knn_lin_oct(f.tree, f.coded, centre, 50, &audit);
                CHECK(nb.size() == 50 && nb[0].dist_sq == 0.0);
                std::printf("[%s] knn_lin_oct %d: %u %.17g %u %.17g\n", cname, i, nb[1].index, nb[1].dist_sq,
                            nb[49].index, nb[49].dist_sq);
            }
            CHECK(audit.emissions > 0);
            CHECK(audit.worst_margin <= 0.0);
        }

        // run_locality (cli.cpp:228-262): index_map = &coded.permutation for the storage order
        for (const std::vector<std::uint32_t>* index_map : {static_cast<const std::vector<std::uint32_t>*>(nullptr),
                                                            &f.coded.permutation}) {
            const LocalityHistogram hist = index_map ? locality_histogram_approx(f.tree, f.coded, 8, 3000, 4, 4, index_map)
                                                     : locality_histogram(f.tree, f.coded, 8, 4, index_map);
            const auto quart = histogram_quantiles(hist);
            std::uint64_t bins = 0;
            for (const auto& [d, c] : hist.bins) bins = mix(mix(bins, d), c);
            std::printf("[%s] locality map=%d: N %" PRIu64 " k %u centres %" PRIu64 " total %" PRIu64
                        " mean %.17g stddev %.17g G1 %.17g Q %.17g %.17g %.17g at0 %" PRIu64 " bins %016" PRIx64 "\n",
                        cname, index_map != nullptr, hist.cloud_size, hist.k, hist.centres, hist.total(), hist.mean(),
                        hist.stddev(), fisher_pearson_skewness(hist), quart[0], quart[1], quart[2], hist.count_at(0),
                        bins);
        }
    }

    // the reference's exception types at its call sites
    auto throws_invalid = [](auto&& fn) {
        try {
            fn();
        } catch (const std::invalid_argument&) {
            return true;
        } catch (...) {
        }
        return false;
    };
    CHECK(throws_invalid([] { reorder_cloud(PointCloud(), Curve::Morton); }));
    CHECK(throws_invalid([] { SearchKernel(KernelShape::Sphere, {0, 0, 0}, 0.0); }));
    CHECK(throws_invalid([] { build_leaves(std::vector<std::uint64_t>{5, 1}, 4); }));
    std::printf("callsite: %s\n", failures == 0 ? "PASS" : "FAIL");
    return failures == 0 ? 0 : 1;
}
