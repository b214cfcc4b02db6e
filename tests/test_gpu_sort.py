"""Onesweep radix sort edge cases (csrc/reorder.cu K3): cloud sizes around the 3072-key tile
boundary (the last tile's pad keys rank after real digit-255 keys), clouds whose codes are mostly
digit 255 in every byte (points packed at the far corner of the cube), coincident-heavy clouds
(long equal-key runs: stability across tiles and the multi-predecessor look-back), and enough
tiles for deep look-back chains.  Codes and permutation must equal the C restatement's
(reorder.cpp:9-89), and the permutation must be numpy's stable argsort of the codes."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

lo = pytest.importorskip("paper_2603_06771_b200.linoct")

TILE = 256 * 12


@pytest.fixture(scope="module")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    return lo.default_context(0)


def far_corner(rng, n):
    # one point at the origin anchors the cube; the rest crowd the opposite corner, so most
    # codes are 0xff... in every byte (digit 255 in every pass) -- the pad keys' digit
    p = 1.0 - rng.random((n, 3)) * 1e-6
    p[0] = 0.0
    return p


def coincident(rng, n):
    base = rng.random((7, 3))
    return base[rng.integers(0, len(base), n)]


@pytest.mark.parametrize("n", [TILE - 1, TILE, TILE + 1, 2 * TILE - 1, 2 * TILE + 1, 5 * TILE + 17])
@pytest.mark.parametrize("kind", ["far_corner", "uniform"])
@pytest.mark.parametrize("curve", [0, 1])
def test_sort_tile_boundaries(ctx, oracle, n, kind, curve):
    rng = np.random.default_rng(n * 7 + curve)
    pts = far_corner(rng, n) if kind == "far_corner" else rng.random((n, 3))
    coded = lo.reorder_cloud(pts, lo.Curve(curve), 21)
    _, codes, perm, _ = oracle.reorder(pts, curve, 21)
    assert np.array_equal(coded.codes, codes)
    assert np.array_equal(coded.permutation, perm)
    raw = codes[np.argsort(perm)]  # codes in input order
    assert np.array_equal(perm, np.argsort(raw, kind="stable"))


@pytest.mark.parametrize("n", [200_003, 1_000_000])
def test_sort_equal_runs_across_many_tiles(ctx, oracle, n):
    rng = np.random.default_rng(n)
    pts = coincident(rng, n)
    coded = lo.reorder_cloud(pts, lo.Curve.Hilbert, 21)
    _, codes, perm, _ = oracle.reorder(pts, 1, 21)
    assert np.array_equal(coded.codes, codes)
    assert np.array_equal(coded.permutation, perm)
