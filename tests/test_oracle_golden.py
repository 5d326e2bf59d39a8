"""The CPU oracle (oracle/) against the golden fixtures frozen from the live
reference: PRNG known answers bit-exact; per-sample step counts, tick stamps
and aggregate counters bit-exact; samples within 1e-12 (BLAS reduction order
differs)."""

import math

import numpy as np
import pytest

from golden_cases import CASES, DEVICE_ONLY, load, oracle_kernel, oracle_target, rel_err, sample_tol, x0_of
from oracle import oracle as O

SAMPLE_TOL = 1e-12


def test_prng_known_answers():
    p = load("prng")
    lib = O.lib()
    for t, b, u, z in zip(p["trip"], p["bits"], p["uniform"], p["normal"]):
        t = [int(v) for v in t]
        assert lib.or_bits(*t) == int(b)
        assert lib.or_uniform(*t) == u
        assert lib.or_normal(*t) == z
    streams = [O.lib().or_split_stream(0, i) for i in range(3)]
    assert streams == [int(s) for s in p["split_streams"][:3]]
    for s, un, nn in zip(p["run_streams"], p["run_uniform"], p["run_normal"]):
        assert np.array_equal(O.fill(5, int(s), 0, un.size, 1), un)
        assert np.array_equal(O.fill(5, int(s), 0, nn.size, 2), nn)


def test_survey_kats():
    # SURVEY.md section 8c values computed from the reference
    lib = O.lib()
    assert lib.or_bits(0, 0, 0) == 0xa59389b7c5f29906
    assert lib.or_uniform(0, 0, 0) == 0.6467825006165618
    assert lib.or_uniform(123, 4, 567) == 0.007978641439848944
    assert lib.or_normal(0, 0, 0) == 0.3766482861700982


@pytest.mark.parametrize("name", sorted(set(CASES) - DEVICE_ONLY))
def test_oracle_matches_reference(name):
    variants, kspec, tspec = CASES[name]
    g = load(name)
    m, n, seed, chunk = (int(g[k]) for k in ("m", "n", "seed", "tick_chunk"))
    kern, targ = oracle_kernel(kspec), oracle_target(tspec)
    x0 = x0_of(g)
    for v in variants:
        if v == "standard":
            r = O.run_standard(kern, targ, m, n, seed, x0=x0)
        else:
            r = O.run_fsm(kern, targ, m, n, seed, variant=v, tick_chunk=chunk, nthreads=4, x0=x0)
        assert np.array_equal(r["iter_counts"], g[v + "_iter_counts"]), v
        for s, mat in r["loop_counts"].items():
            assert np.array_equal(mat, g[f"{v}_loop_{s}"]), (v, s)
        assert r["tick_count"] == int(g[v + "_tick_count"]), v
        assert np.array_equal(r["block_exec_counts"], g[v + "_block_exec_counts"]), v
        if v != "standard":
            assert np.array_equal(r["sample_ticks"], g[v + "_sample_ticks"]), v
            assert r["native_shared_evals"] == int(g[v + "_native_shared_evals"]), v
        assert rel_err(r["samples"], g[v + "_samples"]) <= sample_tol(name), v


def test_oracle_errors_match_reference():
    e = load("errors")
    for v in ("plain", "bundled"):
        with pytest.raises(O.OracleError) as info:
            O.run_fsm(O.drmh(5, 1.0), O.nanband(2, 2.8, math.nan), 6, 400, 3, variant=v)
        assert [info.value.chain, info.value.iteration] == list(e[f"nan_{v}"])
        assert info.value.label == 2   # PROPOSE
    with pytest.raises(O.OracleError) as info:
        O.run_standard(O.drmh(5, 1.0), O.nanband(2, 2.8, math.inf), 6, 400, 3)
    assert [info.value.chain, info.value.iteration] == list(e["inf_standard"])
    with pytest.raises(O.OracleBudget) as info:
        O.run_fsm(O.drmh(10, 0.5), O.gaussian(np.zeros(1), np.eye(1)), 2, 10_000, 7, tick_budget=250)
    r = info.value.result
    assert r["tick_count"] == int(e["budget_tick_count"])
    assert list(r["sample_counts"]) == list(e["budget_sample_counts"])
    assert np.array_equal(r["iter_counts"], e["budget_iter_counts"])


def test_oracle_slice_errors_match_reference():
    e = load("errors_slice")
    for v in ("plain", "bundled"):
        with pytest.raises(O.OracleError) as info:
            O.run_fsm(O.slice_(1.0), O.nanband(1, 2.0, math.nan), 6, 400, 3, variant=v)
        assert [info.value.chain, info.value.iteration] == list(e[f"nan_{v}"])
        assert info.value.label == 7 and str(e[f"nan_{v}_label"]) == "slice"
    with pytest.raises(O.OracleError) as info:
        O.run_standard(O.slice_(1.0), O.nanband(1, 2.0, math.nan), 6, 400, 3)
    assert [info.value.chain, info.value.iteration] == list(e["nan_standard"])


def test_oracle_slice_cap_hits_expansion_budget():
    """slice_cap: the stepping-out budget (3) binds in some samples and EXPAND
    never runs more often than the budget (slice_sampling.py:83-88)."""
    g = load("slice_cap")
    assert g["plain_loop_2"].max() == 3
    assert np.array_equal(g["plain_iter_counts"], g["plain_loop_2"] + g["plain_loop_4"])


def test_oracle_threads_and_shards_are_exact():
    """Chains are independent: threading and chain sharding change nothing."""
    k, t = O.drmh(100, 0.1), O.mog(10, 0.9, [-3.0, 0.0, 3.0])
    full = O.run_fsm(k, t, 24, 60, 11, variant="bundled", nthreads=1)
    thr = O.run_fsm(k, t, 24, 60, 11, variant="bundled", nthreads=6)
    assert np.array_equal(full["samples"], thr["samples"])
    lo = O.run_fsm(k, t, 10, 60, 11, variant="bundled")
    hi = O.run_fsm(k, t, 14, 60, 11, variant="bundled", chain_offset=10)
    assert np.array_equal(np.concatenate([lo["samples"], hi["samples"]], axis=1), full["samples"])
    assert np.array_equal(np.concatenate([lo["sample_ticks"], hi["sample_ticks"]], axis=1),
                          full["sample_ticks"])


def test_oracle_without_surplus_ticks_keeps_every_per_sample_field():
    """run_fsm(surplus=False) (the CPU baseline beside the engine's
    surplus=False bench runs) skips only the ticks chains take after their
    n-th sample: samples, per-sample counts and tick_count are unchanged,
    the aggregate block counts can only shrink."""
    import numpy as np
    from oracle import oracle as O
    k, t = O.drmh(100, 0.1), O.mog(10, 0.9, [-3.0, 0.0, 3.0])
    a = O.run_fsm(k, t, 24, 60, 5, variant="bundled", nthreads=4)
    b = O.run_fsm(k, t, 24, 60, 5, variant="bundled", nthreads=4, surplus=False)
    assert np.array_equal(a["samples"], b["samples"])
    assert np.array_equal(a["iter_counts"], b["iter_counts"])
    assert np.array_equal(a["sample_ticks"], b["sample_ticks"])
    assert a["tick_count"] == b["tick_count"]
    assert (b["block_exec_counts"] <= a["block_exec_counts"]).all()
    assert (b["block_exec_counts"] < a["block_exec_counts"]).any()
