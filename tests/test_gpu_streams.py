"""The edge phase's stream layout never changes a result (DESIGN 2, "Streams").

generate_stats runs its kernels on five streams ordered by events (dense engine beside the slab
join, the global points and the global unit on their own stream during the chain phase, the tail
pairs beside wave 2, wave 2's sort on the side stream). Every A/B switch that restores a one-stream
variant must give the reference's golden result, and so must the default layout, for the counters,
the exact degrees (MODE 1 atomics) and the materialised edges (MODE 2): a missing event shows up
here as a lost or doubled contribution.
"""
import os

import numpy as np
import pytest

import paper_1710_07565_b200 as rhg

pytestmark = pytest.mark.gpu

VARIANTS = [
    {},
    {"RHG_CONCURRENT_ENGINES": "0"},
    {"RHG_SIDE_SMALL": "0"},
    {"RHG_SIDE_SMALL": "1"},
    {"RHG_SIDE_SMALL": "2"},
    {"RHG_GLOB_STREAM": "0"},
    {"RHG_SORT2_SIDE": "0"},
    {"RHG_MAIN_PRIO": "0"},
    {"RHG_DENSE_PRIO": "1"},
    {"RHG_NO_WAVES": "1"},
]


class _Env:
    def __init__(self, env):
        self.env, self.saved = env, {}

    def __enter__(self):
        for k, v in self.env.items():
            self.saved[k] = os.environ.get(k)
            os.environ[k] = v

    def __exit__(self, *a):
        for k, v in self.saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _params(s):
    return rhg.ModelParams(s["n"], s["alpha"], float.fromhex(s["C"]), s["seed"], s["P"])


@pytest.mark.parametrize("env", VARIANTS, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()) or "default")
def test_stream_layouts_equal_golden(golden, env):
    rows = [s for s in golden["stats"] if s["name"] in ("cfg1", "cfg2", "smoke", "odd_P")]
    assert rows
    with _Env(env):
        for s in rows:
            name = s["name"]
            st = rhg.generate_stats(_params(s))
            assert (st.total.edges, st.total.fingerprint, st.total.comps) == (s["edges"], s["fingerprint"],
                                                                               s["comps"]), (name, env)


@pytest.mark.parametrize("env", VARIANTS[:6], ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()) or "default")
def test_stream_layouts_degrees_and_edges(golden, env):
    s = [r for r in golden["stats"] if r["name"] == "cfg1" and r["P"] == 64][0]
    p = _params(s)
    base_deg = rhg.generate_stats(p, degrees=True).degrees
    base_edges, _ = rhg.generate_edges(p)
    with _Env(env):
        for _ in range(3):  # repeated: a race would not show on every run
            deg = rhg.generate_stats(p, degrees=True).degrees
            assert np.array_equal(deg, base_deg), env
            assert int(deg.sum()) == 2 * s["edges"]
        e, _ = rhg.generate_edges(p)
        assert np.array_equal(e, base_edges), env
        assert len(e) == s["edges"]
