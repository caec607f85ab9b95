"""Predicate audit (north_star "borderline pairs"): every pair the slab join's
FP32 pre-filter decides is re-evaluated with the reference predicate (sweep.hpp:531-533);
the device decision must equal the reference's for every pair (disagreements == 0), the
observed pre-filter error must stay inside its bound tau (max_err_over_tau < 1), and the
audited run still returns the reference's golden counters."""
import pytest

import paper_1710_07565_b200 as rhg

pytestmark = pytest.mark.gpu


def _golden(golden, name, P):
    return [s for s in golden["stats"] if s["name"] == name and s["P"] == P][0]


@pytest.mark.parametrize("name,P,world", [("cfg1", 8, 1), ("cfg2", 64, 1), ("cfg3", 512, 1), ("cfg4_1gpu", 4096, 1)])
def test_predicate_audit(golden, name, P, world):
    s = _golden(golden, name, P)
    p = rhg.ModelParams(s["n"], s["alpha"], float.fromhex(s["C"]), s["seed"], s["P"])
    rep, st = rhg.audit_predicate(p)
    assert (st.total.edges, st.total.fingerprint, st.total.comps) == (s["edges"], s["fingerprint"], s["comps"])
    assert rep["disagreements"] == 0, rep
    assert rep["max_err_over_tau"] < 1.0, rep
    assert rep["slab_pairs"] == rep["prefilter_decided"] + rep["exact_recheck"] + rep["exact_only"]
    assert rep["slab_pairs"] + rep["exact_engine_pairs"] == s["comps"]
    assert rep["slab_pairs"] <= st.stream_comps  # the tail kernel evaluates the predicate itself
