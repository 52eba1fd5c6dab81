"""Multi-process (gloo, CPU) tests of the distributed driver's host logic:
flop-balanced row split, block concatenation by all_gather'd nnz counts.
The local multiply and the partition are the oracle's (injected), so no GPU
is needed; the CUDA path of each rank is what the gpu tests check."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class _HostCSR:
    def __init__(self, M):
        self.M = M
        self.nrows, self.ncols = M.nrows, M.ncols


def _worker(rank, world, port, result_dir):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import synth
    from paper_1804_01698_b200 import dist as sdist

    A, B, _ = synth.workload("c3_rmat20", scale=10)
    hA, hB = _HostCSR(A), _HostCSR(B)

    def part(X, Y, n):
        f, tot = oracle.flop(X.M, Y.M)
        return oracle.rows_to_threads(f, n).tolist(), tot

    def local(X, Y, r0, r1, sorted_):
        return oracle.spgemm(X.M, Y.M, r0, r1)

    blk = sdist.spgemm_dist(hA, hB, True, partition=part, local_spgemm=local)
    rp, col, val = blk.C
    np.savez(os.path.join(result_dir, f"r{rank}.npz"), rp=rp, col=col, val=val,
             r0=blk.row_begin, r1=blk.row_end, off=blk.nnz_offset, tot=blk.nnz_total,
             offs=np.array(blk.offsets))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_spgemm_dist_gloo(tmp_path, world):
    import oracle
    import synth
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    A, B, _ = synth.workload("c3_rmat20", scale=10)
    rp, col, val = oracle.spgemm(A, B)
    parts = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    assert parts[0]["r0"] == 0 and parts[-1]["r1"] == A.nrows
    for a, b in zip(parts, parts[1:]):
        assert a["r1"] == b["r0"]
    f, tot = oracle.flop(A, B)
    assert parts[0]["offs"].tolist() == oracle.rows_to_threads(f, world).tolist()
    cat_col = np.concatenate([p["col"] for p in parts])
    cat_val = np.concatenate([p["val"] for p in parts])
    assert all(int(p["tot"]) == len(col) for p in parts)
    off = 0
    for p in parts:
        assert int(p["off"]) == off
        off += int(p["rp"][-1])
    assert (cat_col == col).all() and (cat_val == val).all()
    ps = np.r_[0, np.cumsum(f)]
    work = [ps[int(p["r1"])] - ps[int(p["r0"])] for p in parts]
    assert max(work) <= -(-tot // world) + f.max()
