// C++ shim test: the reference's entry-point shapes (linoct::b200) against brute force, the
// same kinds of checks the reference's own tests make (proj/tests/test_search.cpp,
// test_reorder.cpp, test_linear_octree.cpp), plus the shim's own extensions (CSR batches,
// device-only clouds, PCB1 / LOC1 files).  Built by __graft_entry__.build(); run by
// tests/test_cpp_shim.py.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
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
    {
        std::vector<Point> pts = {{3.5, 7.9, 2.0}, {0, 0, 0}, {8, 8, 8}};
        auto codes = compute_codes(PointCloud(pts), Curve::Morton);
        EXPECT(codes.size() == 3);
        EXPECT(morton_encode({3, 7, 2}, 3) == 190);  // test_sfc.cpp KAT
        EXPECT(hilbert_decode(hilbert_encode({2, 1, 3}, 2), 2) == (GridCell{2, 1, 3}));
    }
    const std::size_t n = 30000;
    std::vector<Point> pts(n);
    EXPECT(lo_generate_uniform(n, 7, 100.0, &pts[0].x) == LO_OK);
    for (Curve curve : {Curve::Morton, Curve::Hilbert}) {
        const CodedCloud coded = reorder_cloud(PointCloud(pts), curve);
        const auto& codes = coded.codes;
        EXPECT(codes.size() == n && std::is_sorted(codes.begin(), codes.end()));
        const auto& perm = coded.permutation;
        const PointCloud& cloud = coded.cloud;
        for (std::size_t i = 0; i < n; i += 37) EXPECT(cloud[i] == pts[perm[i]]);
        auto inv = invert_permutation(perm);
        for (std::size_t i = 0; i < n; i += 41) EXPECT(perm[inv[i]] == i);
        // the discretizer reproduces every code (compute_codes with an explicit Discretizer)
        EXPECT(compute_codes(cloud, curve, coded.discretizer) == codes);
        const LinearOctree tree(coded, 32);
        auto la = build_leaves(codes, 32);
        EXPECT(la.boundaries == tree.leaves().boundaries && la.offsets == tree.leaves().offsets);
        EXPECT(la.boundaries.front() == 0 && la.boundaries.back() == (std::uint64_t{1} << 63));
        // radius: every 997th centre against a scan (oracles.hpp:19-26)
        BatchOptions opt;
        opt.collect_results = true;
        auto res = run_radius_batch(tree, coded, RadiusMethod::Lin, KernelShape::Sphere, 4.0, opt);
        auto csr = run_radius_batch_csr(tree, coded, RadiusMethod::Lin, KernelShape::Sphere, 4.0, opt);
        EXPECT(res.results.size() == n && csr.counts == res.counts && csr.fingerprints == res.fingerprints);
        for (std::size_t q = 0; q < n; q += 997) {
            std::vector<std::uint32_t> want;
            const SearchKernel kernel(KernelShape::Sphere, cloud[q], 4.0);
            for (std::uint32_t i = 0; i < n; ++i)
                if (kernel_contains(kernel, cloud[i])) want.push_back(i);
            EXPECT(res.results[q] == want && csr.row(q) == want);
            EXPECT(neighbours_lin(tree, coded, kernel) == want);
        }
        // kNN vs brute force with the (dist, index) order (oracles.hpp:29-45)
        auto kr = run_knn_batch(tree, coded, 20, opt);
        for (std::size_t q = 0; q < n; q += 1009) {
            std::vector<std::pair<double, std::uint32_t>> all(n);
            for (std::uint32_t i = 0; i < n; ++i) {
                const double dx = cloud[i].x - cloud[q].x, dy = cloud[i].y - cloud[q].y, dz = cloud[i].z - cloud[q].z;
                all[i] = {dx * dx + dy * dy + dz * dz, i};
            }
            std::partial_sort(all.begin(), all.begin() + 20, all.end());
            KnnAudit audit;
            auto one = knn_lin_oct(tree, coded, cloud[q], 20, &audit);
            EXPECT(audit.emissions == 20 && audit.worst_margin <= 0.0);
            for (int j = 0; j < 20; ++j) {
                EXPECT(kr.results[q][j] == all[j].second);
                EXPECT(one[j].index == all[j].second && one[j].dist_sq == all[j].first);
            }
        }
        auto nb = knn_lin_oct(tree, coded, cloud[5], 1);
        EXPECT(nb.size() == 1 && nb[0].dist_sq == 0.0);
        EXPECT(neighbours_prune(tree, coded, SearchKernel(KernelShape::Cube, {50, 50, 50}, 1e5)).size() == n);
        // Struct: ranged rows expand to the Lin rows; a huge kernel contains the root
        auto st = run_radius_batch(tree, coded, RadiusMethod::Struct, KernelShape::Sphere, 4.0, opt);
        EXPECT(st.counts == res.counts && st.results == res.results);
        for (std::size_t q = 0; q < n; q += 1499) {
            auto rr = neighbours_struct(tree, coded, SearchKernel(KernelShape::Sphere, cloud[q], 4.0));
            EXPECT(rr.expand() == res.results[q] && rr.count() == res.counts[q]);
        }
        // RandomSubset: the reference's sampler, including an empty subset (0 rows, not Full)
        BatchOptions sub;
        sub.mode = BatchMode::RandomSubset;
        sub.subset_size = 500;
        sub.seed = 3;
        auto sr = run_radius_batch(tree, coded, RadiusMethod::Lin, KernelShape::Sphere, 4.0, sub);
        EXPECT(sr.centers.size() == 500);
        for (std::size_t i = 0; i < 500; ++i) EXPECT(sr.fingerprints[i] == res.fingerprints[sr.centers[i]]);
        sub.subset_size = 0;
        auto empty = run_radius_batch(tree, coded, RadiusMethod::Lin, KernelShape::Sphere, 4.0, sub);
        EXPECT(empty.centers.empty() && empty.counts.empty() && empty.mean_count == 0.0);
        auto kempty = run_knn_batch(tree, coded, 8, sub);
        EXPECT(kempty.centers.empty() && kempty.counts.empty());
        auto lempty = locality_histogram_approx(tree, coded, 8, 0, 1);
        EXPECT(lempty.centres == 0 && lempty.total() == 0);
        // LOC1 round trip and the LeafArray constructor give the same tree
        const std::string loc = "/tmp/lo_shim_test.loc", pcb = "/tmp/lo_shim_test.pcb";
        tree.serialize(loc);
        auto loaded = LinearOctree::deserialize(loc, coded);
        EXPECT(loaded.leaves().boundaries == tree.leaves().boundaries && loaded.root() == tree.root());
        EXPECT(loaded.internal_nodes().size() == tree.internal_nodes().size());
        const LinearOctree relinked(tree.leaves(), coded.discretizer, curve, 32);
        EXPECT(relinked.internal_nodes().size() == tree.internal_nodes().size() && relinked.root() == tree.root() &&
               std::memcmp(relinked.internal_nodes().data(), tree.internal_nodes().data(),
                           tree.internal_nodes().size() * sizeof(lo_internal_node)) == 0);
        for (int r : {0, 3, 17}) {  // node boxes agree before and after attaching to the cloud
            const auto a = relinked.node_bounds(r), b = tree.node_bounds(r);
            EXPECT(a == b);
        }
        EXPECT(run_radius_batch(relinked, coded, RadiusMethod::Lin, KernelShape::Sphere, 4.0, BatchOptions{}).fingerprints ==
               res.fingerprints);
        write_pcb(coded, pcb);
        auto again = reorder_pcb(pcb, curve);
        again.download_host_fields();
        EXPECT(again.codes == coded.codes);
        auto dev_only = reorder_cloud_device(PointCloud(pts), curve);
        EXPECT(dev_only.codes.empty() && dev_only.size() == n);
        EXPECT(run_knn_batch(LinearOctree(dev_only, 32), dev_only, 20, BatchOptions{}).fingerprints == kr.fingerprints);
        EXPECT(throws<std::runtime_error>([&] { reorder_pcb("/nonexistent/x.pcb", curve); }));
        std::remove(loc.c_str());
        std::remove(pcb.c_str());
        auto hist = locality_histogram(tree, coded, 8);
        EXPECT(hist.total() == 8ull * n && hist.count_at(0) == n);
        auto qs = histogram_quantiles(hist);
        EXPECT(qs[0] <= qs[1] && qs[1] <= qs[2] && hist.stddev() > 0.0 && fisher_pearson_skewness(hist) > 0.0);
        auto mem = measure_structure(tree);
        EXPECT(mem.node_count == tree.node_count() && mem.bytes_total > 0);
        EXPECT(expected_overhead(linear_octree_cost_params(mem.rho())) > 0.0);
        auto all = neighbours_struct(tree, coded, SearchKernel(KernelShape::Sphere, {50, 50, 50}, 1e5));
        EXPECT(all.ranges.size() == 1 && all.ranges[0].first == 0 && all.ranges[0].second == n &&
               all.singles.empty());
    }
    // reference exception types (reorder.cpp:67, search.cpp:192, linear_octree.cpp:25-33,
    // geometry.hpp:66-69 / :108-111, sfc.hpp:105)
    EXPECT(throws<std::invalid_argument>([] { reorder_cloud(PointCloud(), Curve::Morton); }));
    EXPECT(throws<std::invalid_argument>([] { build_leaves({3, 2, 1}, 8); }));
    EXPECT(throws<std::invalid_argument>([] { build_leaves({1, 2, 3}, 0); }));
    EXPECT(throws<std::invalid_argument>([] { PointCloud({{0, 0, 0}, {1, NAN, 0}}); }));
    EXPECT(throws<std::invalid_argument>([] { SearchKernel(KernelShape::Sphere, {0, 0, 0}, -1.0); }));
    EXPECT(throws<std::logic_error>([] { (void)PointCloud().bbox(); }));
    EXPECT(throws<std::domain_error>([] {
        const Discretizer d(Aabb{{0, 0, 0}, {1, 1, 1}});
        (void)d.cell({2, 0, 0});
    }));
    {
        const CodedCloud c = reorder_cloud(PointCloud(pts), Curve::Hilbert);
        const LinearOctree t(c, 32);
        EXPECT(throws<std::invalid_argument>([&] { run_knn_batch(t, c, 0, BatchOptions{}); }));
        EXPECT(throws<std::invalid_argument>(
            [&] { run_radius_batch(t, c, RadiusMethod::Ptr, KernelShape::Sphere, 1.0, BatchOptions{}); }));
        BatchOptions big;
        big.mode = BatchMode::RandomSubset;
        big.subset_size = n + 1;
        EXPECT(throws<std::invalid_argument>(
            [&] { run_radius_batch(t, c, RadiusMethod::Lin, KernelShape::Sphere, 1.0, big); }));
    }
    std::printf("shim_test: PASS\n");
    return 0;
}
