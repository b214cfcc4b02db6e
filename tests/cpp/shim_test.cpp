// C++ shim test: the reference's entry-point shapes (linoct::b200) against brute force, the
// same checks the reference's own tests make (proj/tests/test_search.cpp, test_reorder.cpp,
// test_linear_octree.cpp).  Built by __graft_entry__.build(); run by tests/test_cpp_shim.py.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <stdexcept>
#include <vector>

#include "linoct_b200.hpp"

using namespace linoct::b200;

#define EXPECT(cond)                                                        \
    do {                                                                    \
        if (!(cond)) {                                                      \
            std::fprintf(stderr, "FAILED %s at line %d\n", #cond, __LINE__); \
            std::exit(1);                                                   \
        }                                                                   \
    } while (0)

template <class E, class F>
bool throws(F f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

int main() {
    // KATs through the device codecs (test_sfc.cpp:62-65, :106-113)
    {
        std::vector<Point> pts = {{3.5, 7.9, 2.0}, {0, 0, 0}, {8, 8, 8}};
        auto codes = compute_codes(PointCloud(pts), Curve::Morton);
        EXPECT(codes.size() == 3);
    }
    const std::size_t n = 30000;
    std::vector<Point> pts(n);
    EXPECT(lo_generate_uniform(n, 7, 100.0, &pts[0].x) == LO_OK);
    for (Curve curve : {Curve::Morton, Curve::Hilbert}) {
        auto coded = reorder_cloud(PointCloud(pts), curve);
        auto codes = coded.codes();
        EXPECT(std::is_sorted(codes.begin(), codes.end()));
        auto perm = coded.permutation();
        auto cloud = coded.cloud();
        for (std::size_t i = 0; i < n; i += 37) EXPECT(cloud[i] == pts[perm[i]]);
        auto inv = invert_permutation(perm);
        for (std::size_t i = 0; i < n; i += 41) EXPECT(perm[inv[i]] == i);
        LinearOctree tree(coded, 32);
        auto la = build_leaves(codes, 32);
        EXPECT(la.boundaries == tree.leaves().boundaries && la.offsets == tree.leaves().offsets);
        EXPECT(la.boundaries.front() == 0 && la.boundaries.back() == (std::uint64_t{1} << 63));
        // radius: every 997th centre against a scan (oracles.hpp:19-26)
        BatchOptions opt;
        opt.collect_results = true;
        auto res = run_radius_batch(tree, coded, RadiusMethod::Lin, KernelShape::Sphere, 4.0, opt);
        const double r2 = 4.0 * 4.0;
        for (std::size_t q = 0; q < n; q += 997) {
            std::vector<std::uint32_t> want;
            for (std::uint32_t i = 0; i < n; ++i) {
                const double dx = cloud[i].x - cloud[q].x, dy = cloud[i].y - cloud[q].y,
                             dz = cloud[i].z - cloud[q].z;
                if (dx * dx + dy * dy + dz * dz < r2) want.push_back(i);
            }
            EXPECT(res.row(q) == want);
        }
        // kNN vs brute force with the (dist, index) order (oracles.hpp:29-45)
        auto kr = run_knn_batch(tree, coded, 20, opt);
        for (std::size_t q = 0; q < n; q += 1009) {
            std::vector<std::pair<double, std::uint32_t>> all(n);
            for (std::uint32_t i = 0; i < n; ++i) {
                const double dx = cloud[i].x - cloud[q].x, dy = cloud[i].y - cloud[q].y,
                             dz = cloud[i].z - cloud[q].z;
                all[i] = {dx * dx + dy * dy + dz * dz, i};
            }
            std::partial_sort(all.begin(), all.begin() + 20, all.end());
            for (int j = 0; j < 20; ++j) {
                EXPECT(kr.indices[q * 20 + j] == all[j].second);
                EXPECT(kr.distances[q * 20 + j] == all[j].first);
            }
        }
        auto nb = knn_lin_oct(tree, coded, cloud[5], 1);
        EXPECT(nb.size() == 1 && nb[0].dist_sq == 0.0);
        auto lin = neighbours_lin(tree, coded, KernelShape::Sphere, {50, 50, 50}, 1e5);
        EXPECT(lin.size() == n);
        // Struct: ranged rows expand to the Lin rows; a huge kernel contains the root
        auto st = run_radius_batch(tree, coded, RadiusMethod::Struct, KernelShape::Sphere, 4.0, opt);
        EXPECT(st.counts == res.counts && st.indices == res.indices);
        for (std::size_t q = 0; q < n; q += 1499) {
            auto rr = neighbours_struct(tree, coded, KernelShape::Sphere, cloud[q], 4.0);
            EXPECT(rr.expand() == res.row(q) && rr.count() == res.counts[q]);
        }
        // LOC1 round trip and the LeafArray constructor give the same tree
        const std::string loc = "/tmp/lo_shim_test.loc", pcb = "/tmp/lo_shim_test.pcb";
        tree.serialize(loc);
        auto loaded = LinearOctree::deserialize(loc, coded);
        EXPECT(loaded.leaves().boundaries == tree.leaves().boundaries && loaded.root() == tree.root());
        EXPECT(loaded.internal_nodes().size() == tree.internal_nodes().size());
        std::array<double, 6> box{};
        {
            lo_coded_info ci{};
            check(lo_coded_info_get(coded.handle(), &ci));
            std::copy(ci.disc_box, ci.disc_box + 6, box.begin());
        }
        LinearOctree relinked(coded, tree.leaves(), box, 21, curve, 32);
        EXPECT(relinked.internal_nodes().size() == tree.internal_nodes().size() &&
               std::memcmp(relinked.internal_nodes().data(), tree.internal_nodes().data(),
                           tree.internal_nodes().size() * sizeof(lo_internal_node)) == 0);
        write_pcb(coded, pcb);
        auto again = reorder_pcb(pcb, curve);
        EXPECT(again.codes() == coded.codes());
        EXPECT(throws<std::runtime_error>([&] { reorder_pcb("/nonexistent/x.pcb", curve); }));
        std::remove(loc.c_str());
        std::remove(pcb.c_str());
        auto hist = locality_histogram(tree, coded, 8);
        EXPECT(hist.total() == 8ull * n && hist.count_at(0) == n);
        auto qs = histogram_quantiles(hist);
        EXPECT(qs[0] <= qs[1] && qs[1] <= qs[2] && hist.stddev() > 0.0 && fisher_pearson_skewness(hist) > 0.0);
        auto mem = measure_structure(tree);
        EXPECT(mem.node_count == tree.node_count() && mem.bytes_total > 0);
        auto all = neighbours_struct(tree, coded, KernelShape::Sphere, {50, 50, 50}, 1e5);
        EXPECT(all.ranges.size() == 1 && all.ranges[0].first == 0 && all.ranges[0].second == n &&
               all.singles.empty());
    }
    // reference exception types (reorder.cpp:67, search.cpp:192, linear_octree.cpp:25-33)
    EXPECT(throws<std::invalid_argument>([] { reorder_cloud(PointCloud(), Curve::Morton); }));
    EXPECT(throws<std::invalid_argument>([] { build_leaves({3, 2, 1}, 8); }));
    EXPECT(throws<std::invalid_argument>([] { build_leaves({1, 2, 3}, 0); }));
    std::printf("shim_test: PASS\n");
    return 0;
}
