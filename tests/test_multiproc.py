"""CPU, world_size 2 over gloo: the N>1 path shards rows with no data-path
collective; results assembled from the shards equal the single-process
results, shards tile [0, B) exactly, and the job time is the max over ranks."""
import os
import socket

import numpy as np
import pytest

from paper_2509_08383_b200.workloads import shard_rows


@pytest.mark.parametrize("B,world", [(0, 2), (1, 2), (7, 2), (64, 3), (4096, 8), (5, 8)])
def test_shards_tile_rows(B, world):
    cover = []
    for r in range(world):
        r0, r1 = shard_rows(B, r, world)
        assert 0 <= r0 <= r1 <= B
        cover.extend(range(r0, r1))
    assert cover == list(range(B))
    sizes = [shard_rows(B, r, world)[1] - shard_rows(B, r, world)[0] for r in range(world)]
    assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2509_08383_b200 as pam
    from oracle import oracle as orc
    from paper_2509_08383_b200 import workloads as W
    from paper_2509_08383_b200.dist import init_from_env

    env = init_from_env(backend="gloo")
    x = W.gaussian(10, 777, seed=5)
    r0, r1 = env.shard(10)
    z, am, st = orc.cutmax_batch(x[r0:r1], pam.CutMaxParams().lower(), nthreads=1)
    env.barrier()
    t = env.max_over_ranks(float(rank + 1))       # per-rank "device time"
    rows = env.sum_over_ranks(float(r1 - r0))     # units processed by all ranks
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), z=z, am=am, st=st, r0=r0, r1=r1, t=t, rows=rows)
    env.close()


def test_gloo_world2_shards_match_single_process(tmp_path, orc, pam):
    import torch.multiprocessing as mp
    from paper_2509_08383_b200 import workloads as W

    port = _free_port()
    mp.start_processes(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    x = W.gaussian(10, 777, seed=5)
    z_ref, am_ref, st_ref = orc.cutmax_batch(x, pam.CutMaxParams().lower())
    z = np.zeros_like(z_ref)
    am = np.zeros_like(am_ref)
    for r in range(2):
        d = np.load(tmp_path / f"r{r}.npz")
        z[d["r0"]:d["r1"]] = d["z"]
        am[d["r0"]:d["r1"]] = d["am"]
        assert float(d["t"]) == 2.0          # max over ranks
        assert float(d["rows"]) == 10.0      # whole-job units
    assert np.array_equal(am, am_ref)
    assert np.array_equal(z, z_ref)          # same rows, same oracle -> bit-identical
