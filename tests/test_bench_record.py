"""bench.py's roofline bookkeeping (pure host logic): executed flop counts per kernel kind and the
per-class aggregation of the library's kernel-event records."""

import importlib.util
import os

import pytest


@pytest.fixture(scope="module")
def bench():
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "bench.py")
    spec = importlib.util.spec_from_file_location("bench_module", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_kernel_flops_count_only_executed_tiles(bench):
    M, N, K = 1024, 2048, 4096
    assert bench.kernel_flops("ozaki", (M, N, K)) == 2.0 * M * N * K
    assert bench.kernel_flops("ozaki-matvec-core", (M, N, K)) == 2.0 * M * N * K
    # Gram: tiles touching the upper block triangle; triangular operands: k steps up to the block diagonal
    assert bench.kernel_flops("ozaki-gram", (1024, 1024, K)) == 1024.0 * (1024 + 128) * K
    assert bench.kernel_flops("ozaki-tril", (1024, N, 1024)) == 1024.0 * (1024 + 128) * N
    assert bench.kernel_flops("ozaki-triu", (M, 1024, 1024)) == 1.0 * M * 1024 * (1024 + 64)
    assert bench.kernel_flops("ozaki-gram", (1024, 1024, K)) < bench.kernel_flops("ozaki", (1024, 1024, K))


def test_kernel_classes_aggregate_by_kind_and_shape(bench):
    gram = ("ozaki-gram", (1024, 1024, 1 << 20), 15.0)
    gemm = ("ozaki", (1 << 20, 1024, 1024), 24.0)
    kc = bench.kernel_classes([gram, gemm, gram, gemm, gram, gram], steps=2)
    assert [c["kind"] for c in kc] == ["ozaki-gram", "ozaki"]          # sorted by kernel time: 60 ms, 48 ms
    g = kc[0]
    assert g["launches_per_step"] == 2 and g["ms_per_launch"] == 15.0 and g["ms_per_step"] == 30.0
    fl = bench.kernel_flops(*gram[:2])
    assert g["fp64_equivalent_tflops"] == pytest.approx(fl / 15e-3 / 1e12)
    assert g["int8_tops"] == pytest.approx(bench.OZ_PAIRS * fl / 15e-3 / 1e12)
    assert kc[1]["launches_per_step"] == 1 and kc[1]["ms_per_step"] == 24.0
