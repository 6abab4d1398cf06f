"""CPU, world_size 2 over gloo: sharded batch tracking gathers exactly the
unsharded results (the oracle stands in for each rank's GPU tracker)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1501_06625_b200 import PrecisionMode as PM
from paper_1501_06625_b200 import workloads as W
from paper_1501_06625_b200.multi import shard_range, track_batch_sharded


def test_shard_ranges_cover_once():
    for P in (0, 1, 7, 8192):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                lo, hi = shard_range(P, r, world)
                seen.extend(range(lo, hi))
            assert seen == list(range(P))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_path):
    import torch.distributed as dist
    from oracle.orc import Oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = W.random_system(n=6, degree=3, n_monomials=20, prec=PM.DD, n_paths=9)
    orc = Oracle("restatement")
    orc.set_threads(1)

    def track(starts):
        ends, stats = [], []
        for p in range(starts.shape[0]):
            e, st, _ = orc.track_path(int(w.prec), w.g, w.f, w.gamma, w.k, starts[p], w.params)
            ends.append(e)
            stats.append(st)
        return np.array(ends).reshape((-1,) + w.starts.shape[1:]), stats

    res = track_batch_sharded(track, w.starts, rank, world)
    if rank == 0:
        full = track(w.starts)
        np.savez(out_path, ends=res[0], rows=res[1], ref_ends=full[0],
                 ref_steps=np.array([s.steps for s in full[1]]))
    dist.destroy_process_group()


def test_sharded_batch_equals_unsharded(tmp_path):
    out = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    d = np.load(out)
    assert np.array_equal(d["ends"].view(np.uint64), d["ref_ends"].view(np.uint64))
    assert d["rows"][:, 2].tolist() == d["ref_steps"].tolist()
