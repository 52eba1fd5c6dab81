"""The NCCL path of the distributed driver on one GPU (world size 1): B
broadcast, GPU RowsToThreads split, local block, all_gather of nnz, triangle
all_reduce -- checked against the oracle.  (Multi-rank logic: test_dist_gloo.)"""
import os
import socket

import numpy as np
import pytest

import oracle
import synth
from parity import compare

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


def test_spgemm_dist_nccl_world1(pg):
    import paper_1804_01698_b200 as spg
    from paper_1804_01698_b200 import dist as sdist
    A, B, _ = synth.workload("c3_rmat20", scale=12)
    dA = sdist.broadcast_csr(spg.DeviceCSR.from_host(A))
    blk = sdist.spgemm_dist(dA, dA, sorted=True)
    assert (blk.row_begin, blk.row_end, blk.nnz_offset) == (0, A.nrows, 0)
    g = blk.C.to_host()
    o = oracle.spgemm(A, B)
    assert blk.nnz_total == len(o[1])
    compare(*g, *o, True, "dist world 1")


def test_triangles_dist_nccl_world1(pg):
    import paper_1804_01698_b200 as spg
    from paper_1804_01698_b200 import dist as sdist
    L, U, ex = synth.workload("c5_triangle", scale=11)
    dL, dU, dG = (spg.DeviceCSR.from_host(x) for x in (L, U, ex["G"]))
    want = oracle.triangle_count(L, U, ex["G"])
    assert sdist.triangle_count_dist(dL, dU, dG) == want
    assert sdist.triangle_count_dist(dL, dU, dG, fused=True) == want
    assert sdist.triangle_count_graph_dist(dG) == want            # degree order
    assert sdist.triangle_count_graph_dist(dG, fused=False) == want
    assert spg.triangle_count_graph(dG) == want
