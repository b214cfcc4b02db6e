"""On-disk formats: PCB1 / text XYZ clouds (io.cpp:16-120) and LOC1
trees (linear_octree.cpp:149-190), checked against the reference library's own readers and
writers -- files written by one side are read by the other, bit for bit, and malformed files
fail with the reference's messages.  The host readers run without a GPU; the device paths
(streamed PCB reorder, LOC1 load + device link from a LeafArray) are marked gpu."""
import os

import numpy as np
import pytest

lo = pytest.importorskip("paper_2603_06771_b200.linoct")


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


@pytest.fixture
def pts(oracle):
    p = oracle.gen_terrain(3000, 91, 50.0)
    p[7] = [-0.0, 1e-310, 123456789.123456789]  # signed zero, subnormal, long mantissa
    return p


@pytest.mark.parametrize("ext", [".pcb", ".xyz"])
def test_cloud_files_vs_reference(tmp_path, ref, pts, ext):
    ours, theirs = str(tmp_path / ("ours" + ext)), str(tmp_path / ("theirs" + ext))
    lo.write_cloud(pts, ours)
    ref.write_cloud(pts, theirs)
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    assert np.array_equal(bits(lo.read_cloud(theirs).points), bits(pts))
    assert np.array_equal(bits(ref.read_cloud(ours)), bits(pts))


def test_cloud_file_errors_match_reference(tmp_path, ref, pts):
    good = str(tmp_path / "a.pcb")
    lo.write_cloud(pts, good)
    raw = open(good, "rb").read()
    cases = {
        "magic.pcb": b"PCB2" + raw[4:],
        "count.pcb": raw[:9],
        "trunc.pcb": raw[:12 + 24 * 17 + 5],
        "nan.pcb": raw[:12 + 24 * 5] + np.float64(np.nan).tobytes() + raw[12 + 24 * 5 + 8:],
        "text.xyz": b"# comment\n1 2 3\n\n4 5\n",
        "inf.xyz": b"1 2 3\n4 inf 6\n",
        "extra.xyz": b"1 2 3 4\n",
    }
    for name, data in cases.items():
        path = str(tmp_path / name)
        open(path, "wb").write(data)
        with pytest.raises(RuntimeError) as want:
            ref.read_cloud(path)
        with pytest.raises(lo.FileFormatError) as got:
            lo.read_cloud(path)
        assert str(got.value) == str(want.value), name
    with pytest.raises(lo.InvalidArgument):
        lo.format_from_path("cloud.las")


@pytest.fixture(scope="module")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    return lo.default_context(0)


@pytest.mark.gpu
@pytest.mark.parametrize("curve", [0, 1])
def test_reorder_pcb_streams_file(ctx, tmp_path, ref, oracle, curve):
    p = oracle.gen_mixed(300000, 17)  # > one staging chunk is covered below with a small chunk
    path = str(tmp_path / "c.pcb")
    ref.write_cloud(p, path)
    a = lo.reorder_pcb(path, lo.Curve(curve))
    b = lo.reorder_cloud(p, lo.Curve(curve))
    assert np.array_equal(a.codes, b.codes) and np.array_equal(a.permutation, b.permutation)
    assert np.array_equal(bits(a.cloud.points), bits(b.cloud.points))
    # the sorted cloud written by the device path is what the reference reads back
    out = str(tmp_path / "sorted.pcb")
    a.write_pcb(out)
    assert np.array_equal(bits(ref.read_cloud(out)), bits(b.cloud.points))


@pytest.mark.gpu
def test_reorder_pcb_large_multi_chunk(ctx, tmp_path, oracle):
    p = oracle.gen_uniform(5_000_000, 3, 100.0)  # 120 MB: several 48 MiB staging chunks
    path = str(tmp_path / "big.pcb")
    lo.write_cloud(p, path)
    a = lo.reorder_pcb(path, lo.Curve.Hilbert)
    b = lo.reorder_cloud(p, lo.Curve.Hilbert)
    assert np.array_equal(a.codes, b.codes) and np.array_equal(a.permutation, b.permutation)


@pytest.mark.gpu
def test_reorder_pcb_errors(ctx, tmp_path, pts):
    good = str(tmp_path / "a.pcb")
    lo.write_cloud(pts, good)
    raw = open(good, "rb").read()
    for data, msg in [(b"XXXX" + raw[4:], "bad magic at byte offset 0"),
                      (raw[:12 + 24 * 9 + 3], f"truncated record at byte offset {12 + 24 * 9}"),
                      (raw[:12 + 24 * 4] + np.float64(np.inf).tobytes() + raw[12 + 24 * 4 + 8:],
                       "non-finite coordinate in record 4")]:
        path = str(tmp_path / "bad.pcb")
        open(path, "wb").write(data)
        with pytest.raises(lo.FileFormatError, match=msg):
            lo.reorder_pcb(path, lo.Curve.Morton)


@pytest.mark.gpu
@pytest.mark.parametrize("curve,n_max", [(0, 32), (1, 8), (1, 1)])
def test_loc1_roundtrip_vs_reference(ctx, tmp_path, ref, oracle, curve, n_max):
    p = oracle.gen_terrain(40000, 5 + n_max, 100.0)
    rp = ref.pipeline(p, curve, n_max, threads=4)
    coded = lo.reorder_cloud(p, lo.Curve(curve))
    tree = lo.LinearOctree(coded, n_max)
    ours, theirs = str(tmp_path / "ours.loc"), str(tmp_path / "theirs.loc")
    tree.serialize(ours)
    rp.save_tree(theirs)
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    loaded = lo.LinearOctree.deserialize(theirs, coded)
    b, o, nodes = rp.tree()
    la = loaded.leaves()
    assert np.array_equal(la.boundaries, b) and np.array_equal(la.offsets, o)
    assert loaded.internal_nodes().tobytes() == nodes.tobytes() and loaded.root() == rp.root
    assert loaded.n_max() == n_max
    # searches over the loaded tree equal the reference's
    want = rp.radius(1.5, method=1, threads=8)
    got = lo.run_radius_batch(loaded, coded, lo.RadiusMethod.Lin, lo.KernelShape.Sphere, 1.5, lo.BatchOptions())
    assert np.array_equal(got.counts, want["counts"]) and np.array_equal(got.fingerprints, want["fps"])
    wk = rp.knn(12, threads=8)
    gk = lo.run_knn_batch(loaded, coded, 12, lo.BatchOptions())
    assert np.array_equal(gk.fingerprints, wk["fps"])


@pytest.mark.gpu
def test_from_leaves_arbitrary_tilings(ctx, ref, oracle):
    p = oracle.gen_uniform(20000, 8, 10.0)
    coded = lo.reorder_cloud(p, lo.Curve.Hilbert)
    codes = coded.codes
    L = 21
    rng = np.random.default_rng(4)
    for trial in range(6):
        # random aligned power-of-8 tiling: split blocks at random down to depth <= 6
        blocks = [(0, 0)]
        out = []
        while blocks:
            s, d = blocks.pop()
            if d < 6 and rng.random() < (0.9 if d < 2 else 0.45):
                sub = 1 << (3 * (L - d - 1))
                blocks.extend((s + c * sub, d + 1) for c in reversed(range(8)))
            else:
                out.append(s)
        b = np.array(sorted(out) + [1 << 63], np.uint64)
        o = np.searchsorted(codes, b, side="left").astype(np.uint32)
        rb, ro, rn, rroot = ref.link_tree(b=b, o=o, box=coded.disc_box, level=L, curve=1, n_max=7)
        t = lo.LinearOctree.from_leaves(coded, lo.LeafArray(b, o), coded.disc_box, L, lo.Curve.Hilbert, 7)
        assert t.internal_nodes().tobytes() == rn.tobytes() and t.root() == rroot, trial
        # and the tree searches exactly
        c = coded.cloud.points[::1999]
        for row, q in zip(lo.radius_points(t, coded, lo.KernelShape.Sphere, 0.7, c), c):
            assert np.array_equal(row, oracle.radius_brute(coded.cloud.points, q, 0.7, 0))


@pytest.mark.gpu
def test_from_leaves_validation(ctx, ref, oracle):
    p = oracle.gen_uniform(1000, 9, 10.0)
    coded = lo.reorder_cloud(p, lo.Curve.Morton)
    full = 1 << 63
    box = coded.disc_box
    bad = [
        (np.array([0], np.uint64), np.array([0], np.uint32)),                       # too short
        (np.array([1, full], np.uint64), np.array([0, 1000], np.uint32)),           # front != 0
        (np.array([0, full - 1], np.uint64), np.array([0, 1000], np.uint32)),       # back != 8^L
        (np.array([0, 3, full], np.uint64), np.array([0, 0, 1000], np.uint32)),     # misaligned
        (np.array([0, 1 << 60, full], np.uint64), np.array([0, 0, 1000], np.uint32)),  # not pow8 span
        (np.array([0, 1 << 60, 2 << 60, 3 << 60, 4 << 60, 5 << 60, 6 << 60, 7 << 60, full], np.uint64),
         np.array([0, 5, 4, 100, 200, 300, 400, 500, 1000], np.uint32)),            # offsets decrease
    ]
    for b, o in bad:
        with pytest.raises(ValueError) as want:
            ref.link_tree(b=b, o=o, box=box, level=21, curve=0, n_max=8)
        with pytest.raises(lo.InvalidArgument) as got:
            lo.LinearOctree.from_leaves(coded, lo.LeafArray(b, o), box, 21, lo.Curve.Morton, 8)
        assert str(got.value) == str(want.value)
    # a valid tiling whose offsets do not index this cloud is refused (the device tree searches it)
    with pytest.raises(lo.InvalidArgument, match="does not match"):
        lo.LinearOctree.from_leaves(coded, lo.LeafArray(np.array([0, full], np.uint64),
                                                        np.array([0, 999], np.uint32)), box, 21,
                                    lo.Curve.Morton, 8)
