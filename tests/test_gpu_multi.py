"""Multi-GPU entry points on the one GPU this environment has.

* rhg_create_multi over one device: the whole-graph fan-out / merge and the NCCL
  all-reduce call (ncclCommInitAll over one GPU) run for real and return the reference's
  golden counters;
* rhg_attach_comm (one process per GPU) with world = 1 in a fresh process: the device-side
  ncclAllReduce(uint64) ends every shard call and RunStats.reduced_world reports it.
NCCL cannot place two ranks on one GPU, so world > 1 on hardware needs a multi-GPU box; the
shard arithmetic itself (partial results summing to the whole) is covered by
test_gpu_parity.py::test_shards_sum_to_whole and test_gpu_sampler.py (cfg4/cfg5 shards).
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1710_07565_b200 as rhg

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _golden(golden, name, P=None):
    return [s for s in golden["stats"] if s["name"] == name and (P is None or s["P"] == P)][0]


def test_multi_context_one_device(golden):
    s = _golden(golden, "cfg1", 8)
    p = rhg.ModelParams(s["n"], s["alpha"], float.fromhex(s["C"]), s["seed"], s["P"])
    st = rhg.generate_stats(p, rhg.GenOptions(devices=(0,)))
    assert (st.total.edges, st.total.fingerprint, st.total.comps) == (s["edges"], s["fingerprint"], s["comps"])
    assert st.reduced_world == 1
    single = rhg.generate_stats(p, rhg.GenOptions(device=0), degrees=True)
    multi = rhg.generate_stats(p, rhg.GenOptions(devices=(0,)), degrees=True)
    assert np.array_equal(single.degrees, multi.degrees)
    with pytest.raises(ValueError, match="whole graph"):
        rhg.generate_stats(p, rhg.GenOptions(devices=(0,), rank=0, world=2))


SCRIPT = r"""
import json, sys
sys.path.insert(0, {root!r})
import paper_1710_07565_b200 as rhg
p = rhg.ModelParams({n}, {alpha!r}, float.fromhex({C!r}), {seed}, {P})
uid = rhg.nccl_unique_id()
rhg.attach_comm(1, 0, uid, device=0)
st = rhg.generate_stats(p, rhg.GenOptions(device=0, rank=0, world=1))
print(json.dumps([st.total.edges, st.total.fingerprint, st.total.comps, st.reduced_world]))
"""


def test_attach_comm_world1(golden):
    s = _golden(golden, "cfg1", 8)
    code = SCRIPT.format(root=ROOT, n=s["n"], alpha=s["alpha"], C=s["C"], seed=s["seed"], P=s["P"])
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    got = json.loads(out.stdout.strip().splitlines()[-1])
    assert got == [s["edges"], s["fingerprint"], s["comps"], 1]
