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


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_plan_partitions_the_graph(oracle, world):
    """rhg_shard_extent (host plan, no GPU): the ranks' engine ranges tile [0, P), their owned
    streaming points add up to every streaming point, each rank's halo is the first chunk of
    the next rank's range, and every rank draws all global points (generator.hpp:58-104)."""
    import paper_1710_07565_b200 as rhg
    n, d, alpha, seed, P = 300000, 16.0, 0.8, 3, 16
    p = rhg.ModelParams.from_avg_degree(n, alpha, d, seed, P)
    L = oracle.layout(n, alpha, p.C, seed, P)
    ext = [rhg.shard_extent(p, r, world) for r in range(world)]
    assert ext[0].chunk_begin == 0 and ext[-1].chunk_end == P
    assert all(a.chunk_end == b.chunk_begin for a, b in zip(ext, ext[1:]))
    streaming = L.chunk_counts[L.first_streaming:]
    n_glob = int(L.counts[:L.first_streaming].sum())
    assert sum(e.owned_points for e in ext) == n - n_glob
    for e in ext:
        assert e.global_points == n_glob
        assert e.owned_points == int(streaming[:, e.chunk_begin:e.chunk_end].sum())
        assert e.halo_points == int(streaming[:, e.chunk_end % P].sum())
        assert e.sampled_points == e.owned_points + e.halo_points + e.global_points


def test_shard_plan_rejects_bad_rank():
    import paper_1710_07565_b200 as rhg
    p = rhg.ModelParams.from_avg_degree(1000, 0.8, 8.0, 1, 4)
    with pytest.raises(ValueError, match="rank"):
        rhg.shard_extent(p, 2, 2)
