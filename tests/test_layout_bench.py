"""The layout / traversal study (pkg/src/hitdns/bench.py, kernels.py:236-329) on the GPU.

CPU part: the harness (value generation, packing, statistics, report) and
the oracle restatement of the weight kernel against the reference's own
outputs (tests/golden/bench_weights.npz).  GPU part: hd_bench_weights over
every layout x traversal, bitwise equal to the reference, and the
reference's harness tests (pkg/tests/test_bench.py, test_acceptance.py:214-237).
"""

import os

import numpy as np
import pytest
import torch

from conftest import ROOT

import paper_2211_16718_b200 as hd
from paper_2211_16718_b200 import bench

from oracle import oracle  # noqa: E402  (test infrastructure only)

GOLD = np.load(os.path.join(ROOT, "tests", "golden", "bench_weights.npz"))
COMBOS = [(hd.Layout.INTERLEAVED, "lex"), (hd.Layout.INTERLEAVED, "tiled"),
          (hd.Layout.COMPONENT_CONTIGUOUS, "lex"), (hd.Layout.COMPONENT_CONTIGUOUS, "tiled")]


def test_bytes_per_point_model():
    assert bench.BYTES_PER_POINT == 320


def test_values_match_reference_generator():
    shape = tuple(int(v) for v in GOLD["shape"])
    assert np.array_equal(bench.make_bench_values(shape), GOLD["values"])
    a = bench.make_bench_values(8)
    assert a.shape == ((8 + 2 * bench.X_PAD) * 8 * 8, 5)
    assert np.all(a >= 0.5) and np.all(a < 1.5)


def test_pack_values_permutations():
    vals = np.arange(12.0).reshape(4, 3)
    assert np.array_equal(bench.pack_values(vals, hd.Layout.INTERLEAVED), vals.reshape(-1))
    assert np.array_equal(bench.pack_values(vals, hd.Layout.COMPONENT_CONTIGUOUS), vals.T.reshape(-1))


def test_oracle_weights_match_reference_bitwise():
    nx, ny, nz = (int(v) for v in GOLD["shape"])
    want = oracle.bench_weights(GOLD["values"], nx, ny, nz, bench.X_PAD)
    for layout, trav in COMBOS:
        assert np.array_equal(GOLD[f"out_{int(layout)}_{trav}"], want), (layout, trav)
    assert int(GOLD["wasted_0_tiled"]) == 32 * 8 * 3 - 9 * 5 * 3


def test_record_statistics_and_report():
    rec = bench.BenchRecord(shape=(16, 16, 16), layout=hd.Layout.INTERLEAVED, traversal="lex")
    rec.times = [0.004, 0.002, 0.003]
    assert rec.median_seconds == 0.003 and rec.min_seconds == 0.002
    assert rec.bandwidth_gbs == pytest.approx(4096 * 320 / 0.003 / 1e9, rel=1e-12)
    assert rec.size_label == "16"
    assert bench.BenchRecord((64, 8, 8), hd.Layout.INTERLEAVED, "lex").size_label == "64x8x8"
    soa = bench.BenchRecord((16, 16, 16), hd.Layout.COMPONENT_CONTIGUOUS, "lex", times=[0.006])
    text = bench.bench_report([soa, rec])
    lines = text.splitlines()
    assert lines[0] == "n layout traversal median_s bandwidth_GBs ratio_vs_baseline"
    assert lines[1].endswith(" 2") and lines[2].endswith(" 1")  # baseline = interleaved/lex
    with pytest.warns(RuntimeWarning):
        notes = bench.soft_ordering_checks([rec, soa])
    assert len(notes) == 1


def test_run_case_validates():
    with pytest.raises(ValueError):
        bench.run_case(8, hd.Layout.INTERLEAVED, "spiral")
    with pytest.raises(ValueError):
        bench.run_case(8, hd.Layout.INTERLEAVED, "lex", repeats=0)


@pytest.mark.gpu
def test_gpu_all_combinations_match_reference_bitwise():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    shape = tuple(int(v) for v in GOLD["shape"])
    for layout, trav in COMBOS:
        rec, out = bench.run_case(shape, layout, trav, repeats=1)
        assert np.array_equal(out, GOLD[f"out_{int(layout)}_{trav}"]), (layout, trav)
        assert rec.wasted_lanes == int(GOLD[f"wasted_{int(layout)}_{trav}"])


@pytest.mark.gpu
def test_gpu_ragged_and_wasted_lanes():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    rec, _ = bench.run_case(8, hd.Layout.INTERLEAVED, "tiled", repeats=1)
    assert rec.wasted_lanes == (32 - 8) * 8 * 8 and rec.wasted_fraction == 0.75
    rec64, _ = bench.run_case((64, 8, 8), hd.Layout.INTERLEAVED, "tiled", repeats=1)
    assert rec64.wasted_lanes == 0
    lex, _ = bench.run_case(8, hd.Layout.INTERLEAVED, "lex", repeats=1)
    assert lex.wasted_lanes == 0
    # the paper's ragged 65-wide grid: every combination equal, and equal to the oracle
    shape = (65, 33, 7)
    want = oracle.bench_weights(bench.make_bench_values(shape), *shape, bench.X_PAD)
    for layout, trav in COMBOS:
        _, out = bench.run_case(shape, layout, trav, repeats=1)
        assert np.array_equal(out, want), (layout, trav)


@pytest.mark.gpu
def test_gpu_layout_sweep_table():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    records = bench.layout_sweep(sizes=(16, 32, 48, 64), repeats=2)
    assert len(records) == 8
    lines = bench.bench_report(records).splitlines()
    assert lines[0].startswith("n layout traversal") and len(lines) == 1 + 8 + 1
    import warnings

    with warnings.catch_warnings(record=True) as caught:
        warnings.simplefilter("always")
        notes = bench.soft_ordering_checks(records)
    assert len(caught) == len(notes)
