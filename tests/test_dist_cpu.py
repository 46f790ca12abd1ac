"""Host logic of the row-partitioned (multi-GPU) path on CPU:
world_size-2 gloo process groups exercise the nnz-balanced partition, the
row-block slicing each rank hands to the C ABI, and the NCCL unique-id
broadcast used to join ranks.  No GPU needed (the CUDA path itself is covered
by tests/test_gpu_dist.py with virtual parts and a 1-rank NCCL communicator)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.filterwarnings("ignore::DeprecationWarning")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        from paper_2210_16435_b200 import lib
        from synth import baseline_config
        g, _ = baseline_config(1)
        cuts = lib.partition_rows(g.row_ptr, ws)
        rp, ci, vv, gr = lib.row_block(g.row_ptr, g.col, g.val, g.groups, int(cuts[rank]), int(cuts[rank + 1]))
        blocks = [None] * ws
        dist.all_gather_object(blocks, (int(cuts[rank]), rp, ci, vv, gr))
        # the row blocks tile [0, n) and reassemble W and the groups exactly
        blocks.sort(key=lambda b: b[0])
        rp_all = [np.zeros(1, np.int64)]
        off = 0
        for b in blocks:
            rp_all.append(b[1][1:].astype(np.int64) + off)
            off += int(b[1][-1])
        rp_all = np.concatenate(rp_all)
        ok = (np.array_equal(rp_all, g.row_ptr.astype(np.int64))
              and np.array_equal(np.concatenate([b[2] for b in blocks]), g.col)
              and np.array_equal(np.concatenate([b[3] for b in blocks]), g.val)
              and np.array_equal(np.concatenate([b[4] for b in blocks]), g.groups.astype(np.int32)))
        # unique-id bootstrap: rank 0's 128 bytes reach every rank
        uid = bytes(np.random.default_rng(7).integers(0, 256, 128, dtype=np.uint8)) if rank == 0 else None
        got = lib.broadcast_uid(uid, None)
        ref = bytes(np.random.default_rng(7).integers(0, 256, 128, dtype=np.uint8))
        q.put((rank, bool(ok), got == ref, int(rp[-1]), len(rp) - 1))
    finally:
        dist.destroy_process_group()


def test_partition_and_bootstrap_gloo_ws2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert all(r[1] for r in res), res
    assert all(r[2] for r in res), res
    # nnz-balanced: the two blocks carry similar nnz + 4 rows
    w = [r[3] + 4 * r[4] for r in res]
    assert abs(w[0] - w[1]) <= max(w) * 0.05


def test_partition_rows_properties():
    from paper_2210_16435_b200 import lib
    rng = np.random.default_rng(3)
    deg = rng.pareto(2.5, 1000).astype(np.int64) + 1  # skewed degrees (config-5 style)
    rp = np.concatenate([[0], np.cumsum(deg)]).astype(np.int32)
    for P in (1, 2, 3, 8):
        cuts = lib.partition_rows(rp, P)
        assert cuts[0] == 0 and cuts[-1] == 1000 and np.all(np.diff(cuts) >= 0)
        w = rp.astype(np.int64)[cuts[1:]] - rp.astype(np.int64)[cuts[:-1]] + 4 * np.diff(cuts)
        assert w.max() <= (rp[-1] + 4000) / P + deg.max() + 4
