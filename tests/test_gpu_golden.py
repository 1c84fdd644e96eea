"""Full-plan parity through the DEFAULT path (dedup maps on, leaves sampled without a stored
state) against oracle-written fixtures (tests/golden/*.npz, scripts/make_golden.py, which
imports only oracle/ and workloads/).

Bars (BASELINE north_star): outcomes bit-exact except draws the oracle flags
as lying within 1e-9 of a cumulative-probability boundary (R9); histograms identical
otherwise; amplitudes of dumped leaf states within 1e-10 (fp64).  Sampling P:139 §2.3,
noise after every gate P:173 / P:277, readout P:475.

Also: every noise-draw table and every leaf's u53 uniform of all five configs against the
oracle (exact), the executed work with options.no_dedup = 1 (every instance computed) equal
bit for bit, and the split-level sharding equal to the single run.
"""
import os

import numpy as np
import pytest

import paper_2203_13892_b200.tqsim as T
from oracle import gates as OG
from oracle.noise import noise_codes_np
from oracle.tree import measure_uniform
from tq_testutil import GOLDEN
from workloads import load_config, make_variant

pytestmark = pytest.mark.gpu

AMP_TOL = 1e-10


def golden(name):
    path = os.path.join(GOLDEN, name + ".npz")
    if not os.path.exists(path):
        pytest.fail("missing fixture %s (run scripts/make_golden.py)" % path)
    return np.load(path)


def check_plan(res_plan, z):
    assert res_plan.arity_list == [int(v) for v in z["plan_arities"]]
    assert res_plan.boundary_list == [int(v) for v in z["plan_boundaries"]]


def check_outcomes(leaf_outcomes, z):
    """Golden leaves: outcome bit-exact unless the oracle flagged the draw."""
    leaves = z["leaf"]
    got = np.asarray(leaf_outcomes)[leaves]
    ok = (got == z["outcome"]) | z["flagged"]
    bad = leaves[~ok]
    assert bad.size == 0, ("outcome mismatch", bad[:10].tolist(), got[~ok][:10].tolist(),
                           z["outcome"][~ok][:10].tolist())
    return int(z["flagged"].sum())


def check_leaf_debug(res, z):
    """u53 bit-exact (same keyed Philox, R9), flags equal, totals equal to rounding."""
    leaves = z["leaf"]
    assert np.array_equal(res.leaf_u[leaves], z["u"])
    assert np.array_equal(res.leaf_flagged[leaves], z["flagged"])
    assert np.max(np.abs(res.leaf_total[leaves] - z["total"])) < 1e-11


def check_dumped_amplitudes(n, gates, noise, shots, ar, seed, z, leaves, opts=None):
    L = len(z["plan_arities"])
    res = T.tqsim_run_ex(n, gates, noise, shots, ar, seed, opts, [(L - 1, int(l)) for l in leaves])
    row = {int(l): i for i, l in enumerate(z["chk_leaf"])}
    for i, l in enumerate(leaves):
        c = row[int(l)]
        err = np.max(np.abs(res.dumps[i][z["chk_idx"][c]] - z["chk_amp"][c]))
        assert err <= AMP_TOL, (l, err)
    return res


@pytest.mark.parametrize("cfg,tag", [("c2_qft15", "c2_tree"), ("c3_brick20", "c3_tree")])
def test_full_tree_default_path(cfg, tag):
    """Every leaf of the C2 / C3 tree (10,240) through tqsim_run: outcomes, histogram, u53,
    flags and totals equal the oracle's DFS; amplitudes of every 331st leaf within 1e-10."""
    z = golden(tag)
    w = load_config(cfg)
    n, gates, noise, shots, ar = T.workload_args(w)
    res = T.tqsim_run_ex(n, gates, noise, shots, ar, w.seed, None, (), leaf_debug=True)
    check_plan(res.plan, z)
    assert len(z["leaf"]) == res.plan.n_outcomes
    flagged = check_outcomes(res.leaf_outcomes, z)
    check_leaf_debug(res, z)
    if flagged == 0:
        vals, cnts = np.unique(z["outcome"], return_counts=True)
        assert res.counts == dict(zip(vals.tolist(), cnts.tolist()))
    plain = T.tqsim_run(n, gates, noise, shots, ar, w.seed)           # the north_star call
    assert np.array_equal(plain.leaf_outcomes, res.leaf_outcomes)
    # every instance computed (no shared states): the same outcomes
    nd = T.tqsim_run_ex(n, gates, noise, shots, ar, w.seed, T.default_options(no_dedup=1), leaf_debug=True)
    assert np.array_equal(nd.leaf_outcomes, res.leaf_outcomes)
    assert nd.stats.computed_node_executions == res.plan.node_executions
    assert res.stats.computed_node_executions < res.plan.node_executions
    check_dumped_amplitudes(n, gates, noise, shots, ar, w.seed, z, list(z["chk_leaf"]))


def test_c4_subtrees_default_path():
    """C4 (QAOA-24): 4 complete level-4 subtrees (whole sibling / cousin groups, 128 leaves)
    and one leaf in each of the 16 top-level subtrees, through tqsim_run."""
    z = golden("c4_subtrees")
    w = load_config("c4_qaoa24")
    n, gates, noise, shots, ar = T.workload_args(w)
    res = T.tqsim_run_ex(n, gates, noise, shots, ar, w.seed, None, (), leaf_debug=True)
    check_plan(res.plan, z)
    check_outcomes(res.leaf_outcomes, z)
    check_leaf_debug(res, z)
    T.tqsim_release_run_cache()
    leaves = [int(l) for l in z["chk_leaf"][::9]]
    check_dumped_amplitudes(n, gates, noise, shots, ar, w.seed, z, leaves)
    T.tqsim_release_run_cache()


def test_c5_full_tree_and_shards():
    """C5 (HEA-28, 4 GiB states): the whole 32,768-leaf tree through tqsim_run_ex: every u53
    equals the oracle's, every leaf state has norm 1, the golden sibling pairs (two 8-GPU
    shards) match; then shards 0 and 5 of 8 run through tqsim_execute give the same
    outcomes on their leaf ranges."""
    torch = pytest.importorskip("torch")
    T.tqsim_release_run_cache()
    torch.cuda.empty_cache()
    z = golden("c5_pairs")
    w = load_config("c5_hea28")
    n, gates, noise, shots, ar = T.workload_args(w)
    res = T.tqsim_run_ex(n, gates, noise, shots, ar, w.seed, None, (), leaf_debug=True)
    check_plan(res.plan, z)
    check_outcomes(res.leaf_outcomes, z)
    check_leaf_debug(res, z)
    want_u = np.array([measure_uniform(l, w.seed) for l in range(res.plan.n_outcomes)])
    assert np.array_equal(res.leaf_u, want_u)
    assert np.max(np.abs(res.leaf_total - 1.0)) < 1e-10
    T.tqsim_release_run_cache()
    h = T.tqsim_create(n, gates, noise, shots, ar)
    for rank in (0, 5):
        ws = torch.empty(h.workspace_bytes(rank, 8), dtype=torch.uint8, device="cuda")
        out = torch.zeros(int(h.plan.n_outcomes), dtype=torch.int32, device="cuda")
        h.execute(w.seed, rank, 8, torch.cuda.current_stream().cuda_stream, ws.data_ptr(), ws.numel(),
                  out.data_ptr())
        got = out.cpu().numpy().astype(np.uint32)
        _, _, l0, l1 = T.tqsim_shard_range(h.plan, rank, 8)
        assert np.array_equal(got[l0:l1], res.leaf_outcomes[l0:l1])
        assert not got[:l0].any() and not got[l1:].any()
        del ws
        torch.cuda.empty_cache()
    h.close()


@pytest.mark.parametrize("cfg", ["c1_qft5", "c2_qft15", "c3_brick20", "c4_qaoa24", "c5_hea28"])
def test_all_instance_noise_tables(cfg):
    """The keyed Philox draw of every (gate, node instance) of the tree (row a3) equals the
    oracle's (R1, R7, R8): all levels, all instances."""
    w = load_config(cfg)
    n, gates, noise, shots, ar = T.workload_args(w)
    h = T.tqsim_create(n, gates, noise, shots, ar)
    p = h.plan
    low = OG.lower(gates)
    inst = 1
    for level in range(p.n_levels):
        inst *= p.arities[level]
        b0, b1 = p.boundaries[level], p.boundaries[level + 1]
        got = h.noise_table(w.seed, level, 0, inst)
        g = np.arange(b0, b1)[None, :]
        j = np.arange(inst)[:, None]
        two = np.array([OG.is_two_qubit(low[i]) for i in range(b0, b1)])[None, :]
        want = noise_codes_np(g, j, w.seed, np.where(two, w.p2, w.p1), two)
        assert np.array_equal(got, want), (cfg, level)
    h.close()


@pytest.mark.parametrize("cfg", ["c1_qft5", "c4_qaoa24"])
def test_all_leaf_uniforms(cfg):
    """u53 of every leaf (R9: ctr (0, leaf, 1, 0)) from the device sampler == the oracle's."""
    w = load_config(cfg)
    n, gates, noise, shots, ar = T.workload_args(w)
    res = T.tqsim_run_ex(n, gates, noise, shots, ar, w.seed, None, (), leaf_debug=True)
    want = np.array([measure_uniform(l, w.seed) for l in range(res.plan.n_outcomes)])
    assert np.array_equal(res.leaf_u, want)
    T.tqsim_release_run_cache()


def test_c4_beta0_all_leaves_default_path():
    """C4 with beta = 0: |a_x|^2 = 2^-24 for every trajectory, so C(x) = (x+1) 2^-24 and the
    outcome is floor(u 2^24) except draws the exact R9 rule flags (within 1e-9 of a
    boundary, i.e. frac(u 2^24) 2^-24 < 1e-9 on either side); all 8,192 leaves through
    tqsim_run (dedup maps, no stored leaf states)."""
    w = make_variant("c4_qaoa24_beta0")
    n, gates, noise, shots, ar = T.workload_args(w)
    res = T.tqsim_run_ex(n, gates, noise, shots, ar, w.seed, None, (), leaf_debug=True)
    assert res.plan.n_outcomes == 8192
    assert np.max(np.abs(res.leaf_total - 1.0)) < 1e-10
    band = 1e-9 * 2 ** 24
    flagged = 0
    for l in range(8192):
        v = measure_uniform(l, w.seed) * 2 ** 24
        frac = v - np.floor(v)
        if frac < band or 1.0 - frac < band:
            flagged += 1
            assert res.leaf_flagged[l]
            continue
        assert int(res.leaf_outcomes[l]) == int(np.floor(v)), l
    assert flagged < 0.05 * 8192
    T.tqsim_release_run_cache()


@pytest.mark.parametrize("cfg,worlds", [("c1_qft5", (3, 7, 8)), ("c2_qft15", (3, 8))])
def test_split_level_shards_equal_single_run(cfg, worlds):
    """Sharding below level 0 (W does not divide A_0; ancestors recomputed on
    every shard) gives the single run's outcome array, shard by shard (serial on one GPU)."""
    torch = pytest.importorskip("torch")
    w = load_config(cfg)
    n, gates, noise, shots, ar = T.workload_args(w)
    single = T.tqsim_run(n, gates, noise, shots, ar, 4).leaf_outcomes
    h = T.tqsim_create(n, gates, noise, shots, ar)
    N = int(h.plan.n_outcomes)
    for world in worlds:
        acc = np.zeros(N, dtype=np.int64)
        split, lo, hi = T.tqsim_shard_levels(h.plan, 0, world)
        assert split > 0 or h.plan.arities[0] % world == 0
        for r in range(world):
            ws = torch.empty(h.workspace_bytes(r, world), dtype=torch.uint8, device="cuda")
            o = torch.zeros(N, dtype=torch.int32, device="cuda")
            h.execute(4, r, world, torch.cuda.current_stream().cuda_stream, ws.data_ptr(), ws.numel(),
                      o.data_ptr())
            acc += o.cpu().numpy().astype(np.int64)
        assert np.array_equal(acc.astype(np.uint32), single), world
    h.close()
