"""N>1 host path on CPU: world-size-2 gloo processes, engine shards computed by
the oracle's shard function, reduced by paper_1710_07565_b200.distributed —
must equal the whole-graph result (the device shard arithmetic itself is
tested on the GPU in test_gpu_parity.py::test_shards_sum_to_whole)."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, out):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from oracle.refbind import Oracle
    from paper_1710_07565_b200.distributed import ShardResult, generate_stats_distributed

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, alpha, C, seed, P = cfg
    orc = Oracle()

    def shard_fn(_params, r, w):
        st = orc.generate_stats_shard(n, alpha, C, seed, P, r, w, threads=2)
        return ShardResult(st["edges"], st["fingerprint"], st["comps"], st["seconds"] * 1e3)

    g = generate_stats_distributed(None, rank, world, shard_fn=shard_fn)
    out[rank] = (g.edges, g.fingerprint, g.comps, g.world)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,P", [(2, 8), (2, 5), (3, 7)])
def test_gloo_shards_reduce_to_whole(oracle, world, P):
    n, d, alpha, seed = 40000, 12.0, 0.8, 11
    C = oracle.radial_const_from_avg_degree(d, alpha)
    whole = oracle.generate_stats(n, alpha, C, seed, P, threads=2)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), (n, alpha, C, seed, P), out), nprocs=world, join=True)
    want = (whole["edges"], whole["fingerprint"], whole["comps"], world)
    assert all(out[r] == want for r in range(world)), (dict(out), want)


def test_shard_validation(oracle):
    with pytest.raises(ValueError, match="rank"):
        oracle.generate_stats_shard(1000, 1.0, 1.0, 1, 4, 2, 2)
