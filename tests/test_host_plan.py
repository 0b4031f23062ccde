"""Host-side checks of the C-ABI library (no GPU): exports, validation, level planner, counter law,
residue-class partition.  SURVEY §4 test tiers 1 and 5 (partition arithmetic)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import workloads as W
from paper_2305_11645_b200 import _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rq():
    _build.build()
    import paper_2305_11645_b200 as rq
    return rq


def test_library_exports_every_declared_symbol(rq):
    hdr = open(os.path.join(ROOT, "include", "rqmc.h")).read()
    declared = set(re.findall(r"\b(rqmc_[a-z_]+)\s*\(", hdr))
    assert declared == set(rq.EXPORTS)
    L = C.CDLL(_build.LIB)
    for name in declared:
        assert hasattr(L, name), name


def _plan(rq, **kw):
    base = dict(b=2, m=4, s=4, tau=3, w=[0, 1, 1, 2], z=[1, 1, 3, 1])
    base.update(kw)
    return rq.Plan(**base)


@pytest.mark.parametrize("kw,code", [
    (dict(b=4), "ENOTPRIME"),
    (dict(w=[1, 1, 1, 2]), "EWORDER"),                         # w_1 != 0
    (dict(w=[0, 2, 1, 2]), "EWORDER"),                         # decreasing
    (dict(z=[2, 1, 3, 1]), "EZUNIT"),                          # even z'_1
    (dict(z=[1, 9, 3, 1]), "EZUNIT"),                          # z'_2 >= b^{m-w_2}
    (dict(shift=[0.0, 1.0, 0.5, 0.5]), "ESHIFT"),
    (dict(m=40), "EUNSUPPORTED"),
    (dict(m=33), "EUNSUPPORTED"),          # N = 2^33 > 2^32
    (dict(world=3, rank=3), "EINVAL"),                          # rank outside [0, world)
    (dict(world=17), "EUNSUPPORTED"),                          # more ranks than points (N = 16)
    (dict(s=0, w=[], z=[]), "EDIM"),
])
def test_validation_codes(rq, kw, code):
    with pytest.raises(rq.RqmcError) as ei:
        _plan(rq, **kw)
    assert ei.value.name == code


def test_net_validation(rq):
    m = 4
    ident = [1 << (m - 1 - q) for q in range(m)]
    # coordinate 2 with w=1 may not depend on digit 3 (column deletion)
    full = [8, 12, 14, 15]
    with pytest.raises(rq.RqmcError) as ei:
        rq.Plan(2, m, 2, 2, [0, 1], kind=rq.DIGITAL_NET, C_words=ident + full)
    assert ei.value.name == "ENETMAT"
    # row zeroing removes low bits first: full[3] = 15 -> row-zeroed 14, still non-zero
    ok = [8, 12, 14, 0]
    rq.Plan(2, m, 2, 2, [0, 1], kind=rq.DIGITAL_NET, C_words=ident + ok)
    with pytest.raises(rq.RqmcError) as ei:
        rq.Plan(2, m, 2, 2, [0, 1], kind=rq.DIGITAL_NET, C_words=ident + [16, 0, 0, 0])
    assert ei.value.name == "ENETMAT"


def test_rowzero_net_plan(rq):
    """RQMC_DIGITAL_NET_ROWS (Alg. 3/4): any C accepted (no column deletion), every
    coordinate j <= s* in one dense level of N rows, j > s* dropped (unshifted) or the constant level m
    (shifted); MACs = N s* tau (Alg. 4's additions); b = 3 and words >= 2^m rejected."""
    m = 4
    ident = [1 << (m - 1 - q) for q in range(m)]
    full = [8, 12, 14, 15]
    p = rq.Plan(2, m, 3, 5, [0, 1, 4], kind=rq.DIGITAL_NET_ROWS, C_words=ident + full + full)
    assert [(L["w"], L["j_lo"], L["s_w"], L["M"]) for L in p.levels()] == [(0, 0, 2, 16)]
    assert p.summary()["s_star"] == 2
    assert p.stats()["macs"] == 16 * 2 * 5
    p = rq.Plan(2, m, 3, 5, [0, 1, 4], kind=rq.DIGITAL_NET_ROWS, C_words=ident + full + full, dshift=[1, 2, 3])
    assert [(L["w"], L["j_lo"], L["s_w"], L["M"]) for L in p.levels()] == [(4, 2, 1, 1), (0, 0, 2, 16)]
    with pytest.raises(rq.RqmcError) as ei:
        rq.Plan(3, m, 2, 2, [0, 1], kind=rq.DIGITAL_NET_ROWS, C_words=ident + full)
    assert ei.value.name == "EUNSUPPORTED"
    with pytest.raises(rq.RqmcError) as ei:
        rq.Plan(2, m, 2, 2, [0, 1], kind=rq.DIGITAL_NET_ROWS, C_words=ident + [16, 0, 0, 0])
    assert ei.value.name == "ENETMAT"


def test_level_table_tau_I(rq):
    """w = (0,0,1,2,2), m = 3 -> tau_0=2, tau_1=1, tau_2=2."""
    p = rq.Plan(2, 3, 5, 4, [0, 0, 1, 2, 2], z=[1, 3, 1, 1, 1])
    lv = p.levels()
    assert [(L["w"], L["s_w"], L["j_lo"], L["M"]) for L in lv] == [(2, 2, 3, 2), (1, 1, 2, 4), (0, 2, 0, 8)]
    assert [L["parent"] for L in lv] == [-1, 0, 1]
    assert p.summary()["s_star"] == 5


def test_zero_columns_and_shift_level(rq):
    """Columns j > s* are zero and dropped; with a shift they are the constant row
    phi_j(Delta_j), kept as a 1-row level m (reading C-4)."""
    w = [0, 1, 3, 5, 9]
    p = rq.Plan(2, 3, 5, 2, w, z=[1, 1, 1, 1, 1])
    assert [L["w"] for L in p.levels()] == [1, 0]
    assert p.summary()["s_star"] == 2
    ps = rq.Plan(2, 3, 5, 2, w, z=[1, 1, 1, 1, 1], shift=[0.1] * 5)
    assert [(L["w"], L["s_w"], L["M"]) for L in ps.levels()] == [(3, 3, 1), (1, 1, 4), (0, 1, 8)]
    # unshifted but mapped: Phi^-1 of the zero column is the zero-rule constant, not 0
    pm = rq.Plan(2, 3, 5, 2, w, z=[1, 1, 1, 1, 1], map=rq.MAP_INVNORM)
    assert [(L["w"], L["s_w"], L["M"]) for L in pm.levels()] == [(3, 3, 1), (1, 1, 4), (0, 1, 8)]


def test_counter_law(rq):
    """MACs = tau * sum_{j<=s*} b^{m-w_j} (SPEC S:223 counter law)."""
    for cfg in ("C1", "C2", "C3", "C4"):
        prob = W.make_config(cfg)
        p = rq.Plan.from_problem(prob)
        exp = prob.tau * sum(prob.b ** (prob.m - min(int(wj), prob.m)) for wj in prob.w if wj < prob.m)
        assert p.stats()["macs"] == exp
    p = rq.Plan(2, 24, 4096, 2048, W.w_log(2, 24, 4096), z=np.ones(4096, np.uint64))
    assert p.stats()["macs"] == 2048 * (12 * 2 ** 24 + 4096)       # 4.12e11
    assert p.levels()[p.summary()["checkpoint"]]["w"] == 6          # fused levels 0..5
    assert p.summary()["n_fine"] == 6 and p.summary()["n_bundles"] == 2 ** 18 // 32


def test_all_w_zero_is_dense(rq):
    """All w_j = 0: one level, the dense product."""
    p = rq.Plan(2, 6, 5, 3, [0] * 5, z=[1, 3, 5, 7, 9])
    assert len(p.levels()) == 1 and p.stats()["macs"] == 64 * 5 * 3


@pytest.mark.parametrize("b,m,G", [(2, 8, 2), (2, 8, 4), (2, 8, 8), (3, 5, 3), (3, 5, 9)])
def test_residue_partition_covers_once(rq, b, m, G):
    """Rank g owns k = g (mod G); the union over ranks covers 0..N-1 exactly once."""
    s = 2 * m
    w = W.w_log(b, m, s)
    z = W.draw_z(3, b, m, w)
    seen = np.zeros(b ** m, dtype=np.int64)
    for g in range(G):
        p = rq.Plan(b, m, s, 4, w, z=z, rank=g, world=G)
        nl = p.summary()["N_local"]
        assert nl == b ** m // G
        ks = np.array([p.global_row(i) for i in range(nl)])
        assert np.all(ks % G == g)
        seen[ks] += 1
        for L in p.levels():
            assert L["M_local"] == max(L["M"] // G, 1)
    assert np.all(seen == 1)


@pytest.mark.parametrize("b,m,G", [(3, 6, 2), (3, 6, 4), (3, 6, 8), (2, 9, 3), (2, 9, 6), (5, 4, 2),
                                   (3, 12, 8), (3, 3, 5)])
def test_grouped_partition_covers_once(rq, b, m, G):
    """world not a power of b (b = 3 on 2/4/8 GPUs, ...): ncls = b^gamma >= 32 G classes (gamma <= m) in
    contiguous groups per rank; local row i is k = c0 + (i mod nc) + ncls (i div nc).  The ranks cover
    0..N-1 exactly once, group sizes differ by at most one class, and each level's local rows are
    nc M / ncls (nc replicated rows when M < ncls)."""
    s = 2 * m
    w = W.w_log(b, m, s)
    z = W.draw_z(3, b, m, w)
    N = b ** m
    seen = np.zeros(N, dtype=np.int64)
    sizes = []
    for g in range(G):
        p = rq.Plan(b, m, s, 4, w, z=z, rank=g, world=G)
        pt = p.partition()
        ncls, c0, nc = pt["classes"], pt["first"], pt["count"]
        assert ncls == min(b ** m, next(b ** e for e in range(64) if b ** e >= 32 * G))
        assert c0 == ncls * g // G and nc == ncls * (g + 1) // G - c0 >= 1
        sizes.append(nc)
        ks = p.global_rows()
        assert len(ks) == p.summary()["N_local"] == nc * (N // ncls)
        assert all(p.global_row(i) == ks[i] for i in (0, 1, len(ks) - 1))
        assert np.all((ks % ncls >= c0) & (ks % ncls < c0 + nc))
        seen[ks] += 1
        for L in p.levels():
            assert L["M_local"] == (nc * (L["M"] // ncls) if L["M"] >= ncls else nc)
    assert np.all(seen == 1) and max(sizes) - min(sizes) <= 1


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    import oracle
    import paper_2305_11645_b200 as rq
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    prob = W.make_random(77, 2, 9, 40, 6, shifted=True, mapping=W.MAP_INVNORM)
    p = rq.Plan.from_problem(prob, rank=rank, world=world)
    ks = [p.global_row(i) for i in range(p.summary()["N_local"])]
    part = torch.tensor([oracle.neumaier(oracle.f_rows(prob, ks))], dtype=torch.float64)
    dist.all_reduce(part)                     # the path's one collective
    q.put((rank, float(part.item()) / prob.N))
    dist.destroy_process_group()


def test_gloo_world2_partition_allreduce(rq):
    """world_size-2 gloo run of the N>1 host path: each rank sums f over its residue class (via the
    oracle on CPU), one all_reduce combines them; equals the world=1 Q_N."""
    import multiprocessing as mp
    import socket
    import oracle
    sck = socket.socket()
    sck.bind(("127.0.0.1", 0))
    port = sck.getsockname()[1]
    sck.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for pr in procs:
        pr.join(timeout=60)
    prob = W.make_random(77, 2, 9, 40, 6, shifted=True, mapping=W.MAP_INVNORM)
    full = oracle.qn_sum(prob) / prob.N
    assert abs(res[0] - full) <= 1e-13 * abs(full) and res[0] == res[1]


# ------------------------------------------------------------------ reduced MC and batch layouts (host)

def test_reduced_mc_plan(rq):
    """Reduced MC: no generating vector; shifts rejected; coordinates with w_j >= m keep
    one i.i.d. draw each (N_j = 1: a 1-row level m, P:981 N_{s+1} = 1)."""
    p = rq.Plan(2, 4, 5, 3, [0, 1, 1, 4, 6], kind=rq.REDUCED_MC, seed=5)
    lv = p.levels()
    assert [L["w"] for L in lv] == [4, 1, 0] and [L["s_w"] for L in lv] == [2, 2, 1]
    assert lv[0]["M"] == 1
    with pytest.raises(rq.RqmcError) as ei:
        rq.Plan(2, 4, 3, 3, [0, 1, 1], kind=rq.REDUCED_MC, shift=[0.1, 0.2, 0.3])
    assert ei.value.name == "ESHIFT"


def test_batch_layout_and_workspace(rq):
    """replicas add parallelism, so a batch may fuse more fine levels than a
    single run (C2, tau = 256 < 1024: at most 4 fused levels); the batch workspace covers R replica
    slices."""
    prob = W.make_config("C2")
    pl = rq.Plan.from_problem(prob)
    one = pl.summary()
    deep = pl.summary_batch(64, W.F_EXP_MEAN)
    assert deep["n_fine"] >= one["n_fine"] and deep["n_bundles"] * 64 >= 148
    assert deep["n_fine"] == 4 and pl.summary_batch(64, W.F_CALL_MEAN_EXP) == deep
    c1 = rq.Plan.from_problem(W.make_config("C1"))   # N = 1024: single runs stay coarse
    assert c1.summary()["n_fine"] == 0 and c1.summary_batch(64, W.F_EXP_MEAN)["n_fine"] == 4
    assert pl.summary_batch(1, W.F_EXP_MEAN)["checkpoint"] == one["checkpoint"]
    assert pl.workspace_size_batch(16) >= 16 * pl.workspace_size_batch(1) // 2
    assert pl.workspace_size_batch(16) > pl.workspace_size_batch(1)


def test_run_call_validation(rq):
    """Run-call argument checks of the C ABI return their status before any device work (rqmc.h):
    workspace below rqmc_workspace_size -> EINVAL, lda/ldy < tau -> EDIM, missing / bad f -> EINVAL,
    f without a host f-sum slot or no Y (rqmc_xa_host) -> EINVAL, batch shift outside [0,1) -> ESHIFT, unshifted plan for a lattice batch -> EINVAL, bad level ->
    EINVAL.  Fake non-null pointers are never dereferenced on these paths."""
    L = rq.lib()
    p = _plan(rq, shift=[0.1, 0.2, 0.3, 0.4])
    need = p.workspace_size()
    fake = C.c_void_p(0x1000)
    fs = C.c_void_p(0x2000)
    fp = (C.c_double * 2)(0.2, 1.0)
    st = C.c_void_p(0)
    assert L.rqmc_xa(p._h, fake, 3, fake, 3, 0, fp, fs, fake, need - 1, st) == 1        # EINVAL
    assert L.rqmc_xa(p._h, fake, 2, fake, 3, 0, fp, fs, fake, need, st) == 7            # EDIM (lda)
    assert L.rqmc_xa(p._h, fake, 3, fake, 2, 0, fp, fs, fake, need, st) == 7            # EDIM (ldy)
    assert L.rqmc_qn(p._h, fake, 3, -1, fp, fs, fake, need, st) == 1                    # EINVAL (no f)
    assert L.rqmc_qn(p._h, fake, 3, 9, fp, fs, fake, need, st) == 1                     # EINVAL (bad f)
    assert L.rqmc_qn(p._h, fake, 3, 1, None, fs, fake, need, st) == 1                   # CALL needs fparam
    bad = (C.c_double * 8)(*([0.5] * 7 + [1.0]))
    assert L.rqmc_qn_batch(p._h, 2, bad, None, None, fake, 3, 0, fp, fs, fake, 1 << 30, st) == 5  # ESHIFT
    q = _plan(rq)                                                                        # unshifted
    ok = (C.c_double * 8)(*([0.5] * 8))
    assert L.rqmc_qn_batch(q._h, 2, ok, None, None, fake, 3, 0, fp, fs, fake, 1 << 30, st) == 1   # EINVAL
    assert L.rqmc_points(p._h, 99, 0, 1, None, None, st) == 1                           # EINVAL (level)
    hA = C.cast(C.c_void_p(0x3000), C.POINTER(C.c_double))                           # rqmc_xa_host
    hs = C.cast(C.c_void_p(0x4000), C.POINTER(C.c_double))
    assert L.rqmc_xa_host(p._h, hA, 3, fake, 3, 0, fp, hs, fake, need - 1, st) == 1    # EINVAL (workspace)
    assert L.rqmc_xa_host(p._h, hA, 2, fake, 3, 0, fp, hs, fake, need, st) == 7        # EDIM (lda)
    assert L.rqmc_xa_host(p._h, hA, 3, fake, 2, 0, fp, hs, fake, need, st) == 7        # EDIM (ldy)
    assert L.rqmc_xa_host(p._h, hA, 3, None, 3, 0, fp, hs, fake, need, st) == 1        # EINVAL (no Y)
    assert L.rqmc_xa_host(p._h, hA, 3, fake, 3, 0, fp, None, fake, need, st) == 1      # EINVAL (f, no h_fsum)
    assert L.rqmc_qn_host(p._h, hA, 3, -1, fp, hs, fake, need, st) == 1                # EINVAL (no f)


def test_fine_dispatch_table(rq, monkeypatch):
    """Host-only: every fused-fine parity case of tests/test_gpu_fine_paths.py plans the kernel template
    and fused depth it is meant to cover (rqmc_plan_dispatch; DESIGN.md §7 "Dispatch coverage")."""
    from test_gpu_fine_paths import CASES, RANK_CASES, make_prob
    for cid, (b, m, s, tau, wmode, kind, mapping, ck, nt, tmpl, nf) in CASES.items():
        monkeypatch.setenv("RQMC_CKPT_W", ck)
        monkeypatch.setenv("RQMC_NO_TREE", "1" if nt else "0")
        prob = make_prob(500 + sum(map(ord, cid)), b, m, s, tau, wmode, kind=kind, mapping=mapping)
        pl = rq.Plan.from_problem(prob)
        assert pl.summary()["n_fine"] == nf, cid
        assert pl.dispatch(W.F_EXP_MEAN, want_y=False).startswith(tmpl), (cid, pl.dispatch(W.F_EXP_MEAN))
    for cid, G, ck, tmpl, nf in RANK_CASES:
        b, m, s, tau, wmode, kind, mapping, _, nt, _, _ = CASES[cid]
        monkeypatch.setenv("RQMC_CKPT_W", ck)
        monkeypatch.setenv("RQMC_NO_TREE", "1" if nt else "0")
        prob = make_prob(700 + sum(map(ord, cid)) + G, b, m, s, tau, wmode, kind=kind, mapping=mapping)
        for g in range(G):
            pl = rq.Plan.from_problem(prob, rank=g, world=G)
            assert pl.summary()["n_fine"] == nf and pl.dispatch(W.F_MEAN).startswith(tmpl), (cid, G, g)


def test_batch_chunk_fits_workspace(rq):
    """a tight workspace makes rqmc_qn_batch re-plan its chunk / layout; whatever it picks
    must fit the caller's bytes (the call validates before launching: on a host without a device it
    gets as far as the upload and fails with ECUDA, never EINVAL for a workspace that holds one
    replica)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("host-only check (passes placeholder device pointers)")
    prob = W.make_random(5, 2, 14, 100, 40, shifted=True, mapping=W.MAP_INVNORM)
    pl = rq.Plan.from_problem(prob)
    one, many = pl.workspace_size_batch(1), pl.workspace_size_batch(64)
    assert many > one
    lib = rq.lib()
    sh = np.random.default_rng(0).random((64, prob.s))
    out = (C.c_double * 64)()
    for wb in (one, (one + many) // 3, many - 8, many):
        st = lib.rqmc_qn_batch(pl._h, 64, sh.ctypes.data_as(C.POINTER(C.c_double)), None, None,
                               C.c_void_p(1 << 20), prob.tau, W.F_EXP_MEAN, None,
                               C.cast(out, C.c_void_p), C.c_void_p(1 << 30), wb, None)
        assert st in (0, 9), (wb, st)              # RQMC_OK on a GPU would need real buffers; ECUDA here
    st = lib.rqmc_qn_batch(pl._h, 64, sh.ctypes.data_as(C.POINTER(C.c_double)), None, None,
                           C.c_void_p(1 << 20), prob.tau, W.F_EXP_MEAN, None, C.cast(out, C.c_void_p),
                           C.c_void_p(1 << 30), 4096, None)
    assert st == 1                                 # EINVAL: below one replica of any layout
