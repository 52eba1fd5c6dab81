"""Full-size parity of the BASELINE configs (GPU, marker `gpu` + `slow`).

Expected values come only from the oracle: either computed live here, or
from ``tests/golden/full_configs.json`` written by ``tools/oracle_goldens.py``
(which calls only ``oracle/``).  SURVEY.md §8(c) parity protocol items 1, 4:
row_ptr exact on every row (sha256 of the per-row nnz against the oracle's),
C4 element-wise, C5 triangle count exact three ways (C formed in row blocks,
fused mask, degree order).  C3's values: sampled rows element-wise and the
row-sum identity in test_gpu_parity.py; the streamed all-rows comparison is
``tools/parity_full.py`` (log in profiles/)."""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle
import synth
from parity import compare

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "full_configs.json")))


def _sha(nnz) -> str:
    return hashlib.sha256(np.ascontiguousarray(nnz, dtype="<i8").tobytes()).hexdigest()


@pytest.fixture(scope="module")
def spg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1804_01698_b200 as m
    from paper_1804_01698_b200 import build
    build.build()
    return m


@pytest.fixture(scope="module")
def ctx(spg):
    return spg.Context()


@pytest.fixture(scope="module")
def rmat_sym():
    """C4 / C5 inputs (one R-MAT draw, shared)."""
    return {"c4": synth.workload("c4_tallskinny"), "c5": synth.workload("c5_triangle")}


@pytest.mark.parametrize("name", ["c1_er4096", "c2_stencil64", "c3_rmat20"])
def test_row_structure_all_rows(spg, ctx, name):
    """C.row_ptr of the full-size product equals the oracle's on EVERY row
    (symbolic phase; sha256 of per-row nnz vs the oracle golden)."""
    A, B, _ = synth.workload(name)
    g = GOLD[name]
    dA = spg.DeviceCSR.from_host(A)
    dB = dA if B is A else spg.DeviceCSR.from_host(B)
    rp, nnz, flop = spg.spg_symbolic(dA, dB, ctx)
    assert flop == g["flop"] and nnz == g["nnz_C"]
    assert _sha(np.diff(rp.cpu().numpy())) == g["row_nnz_sha256"]
    info = ctx.info()
    assert info["max_row_flop"] == g["max_row_flop"] and info["max_row_nnz"] == g["max_row_nnz"]


@pytest.mark.parametrize("sorted_out", [False, True])
def test_c4_full_elementwise(spg, ctx, rmat_sym, sorted_out):
    """BASELINE config 4 at full size: whole product vs the oracle."""
    A, B, _ = rmat_sym["c4"]
    dA, dB = spg.DeviceCSR.from_host(A), spg.DeviceCSR.from_host(B)
    C = spg.spgemm(dA, dB, sorted=sorted_out, ctx=ctx)
    o = oracle.spgemm(A, B)
    compare(*C.to_host(), *o, sorted_out, f"C4 full sorted={sorted_out}")
    assert int(o[0][-1]) == GOLD["c4_tallskinny"]["nnz_C"]


def test_c5_full_structure(spg, ctx, rmat_sym):
    """C5's L*U (232 GB, never formed whole): row_ptr of every row vs the oracle."""
    L, U, _ = rmat_sym["c5"]
    dL, dU = spg.DeviceCSR.from_host(L), spg.DeviceCSR.from_host(U)
    rp, nnz, flop = spg.spg_symbolic(dL, dU, ctx)
    g = GOLD["c5_triangle"]
    assert flop == g["flop"] and nnz == g["nnz_C"]
    assert _sha(np.diff(rp.cpu().numpy())) == g["row_nnz_sha256"]


@pytest.mark.parametrize("way", ["formed_sorted", "formed_unsorted", "fused", "degree_order"])
def test_c5_full_triangles(spg, ctx, rmat_sym, way):
    """BASELINE config 5 at full size: the triangle count equals the oracle's
    (natural order, Sec 5.6) whichever GPU path computes it."""
    L, U, ex = rmat_sym["c5"]
    G = ex["G"]
    want = GOLD["c5_triangle"]["triangles"]
    dL, dU, dG = (spg.DeviceCSR.from_host(x) for x in (L, U, G))
    if way.startswith("formed"):
        got = spg.triangle_count(dL, dU, dG, sorted=(way == "formed_sorted"), ctx=ctx)
    elif way == "fused":
        got = spg.triangle_count_fused(dL, dU, dG, ctx=ctx)
    else:
        got = spg.triangle_count_graph(dG, degree_order=True, fused=True, ctx=ctx)
    assert got == want
