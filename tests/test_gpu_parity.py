"""T3/T4 — the CUDA path (through the C ABI) vs the fp64 oracle, on the same seeded inputs.

Tolerances: tests/parity.py (log posteriors and log Z within 1e-9 absolute;
MAP / events exact outside MAP margins < 1e-6 and |p_new - theta| < 1e-6).
Metamorphic checks (chunk split, series permutation, host vs device input)
are bit-exact.
"""
import numpy as np
import pytest

from tests import bruteforce, parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - collected on CPU boxes too
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2410_12588_b200 import bocd, tracegen  # noqa: E402


def _run_gpu(x, R, H, mode, chunks=None, kappa0=1.0, alpha0=1.0, mu0=None, beta0=None,
             prior_cov=0.05, ev_mask=1, cap=64, schedule="auto", threshold=0.9):
    S, T = x.shape
    first = mu0 is None
    b = bocd.BocdBatch(S, R=R, hazard=H, kappa0=kappa0, alpha0=alpha0,
                       mu0=0.0 if first else mu0, beta0=1.0 if first else beta0,
                       prior_first_obs=first, prior_cov=prior_cov, trunc_mode=mode,
                       event_mask=ev_mask, event_capacity=cap, threshold=threshold)
    b.set_schedule(schedule)
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    chunks = chunks or [T]
    maps, pn, lz = [], [], []
    t0 = 0
    for n in chunks:
        m, p, z = b.update_chunk(xd[:, t0:t0 + n], outputs=True)
        maps.append(m.cpu().numpy()); pn.append(p.cpu().numpy()); lz.append(z.cpu().numpy())
        t0 += n
    assert t0 == T
    logR, mu, be = (a.cpu().numpy() for a in b.read_posterior())
    ev, dropped = b.changepoints()
    b.close()
    return dict(map=np.concatenate(maps, 1), pnew=np.concatenate(pn, 1), logz=np.concatenate(lz, 1),
                logR=logR, mu=mu, beta=be, events=ev, dropped=dropped)


def _oracle(oracle_mod, x, R, H, mode, mu0=None, beta0=None, prior_cov=0.05, kappa0=1.0,
            alpha0=1.0, traj=False, threshold=0.9):
    first = mu0 is None
    return oracle_mod.run(x, R, H, kappa0, alpha0, mu0, beta0, trunc_mode=mode, threshold=threshold,
                          prior_first_obs=first, prior_cov=prior_cov, traj=traj, n_threads=0)


def _full_check(g, res, theta=0.9, mask=1, name=None):
    st = parity.compare_steps(g["map"], g["pnew"], g["logz"], res, theta)
    st["max_dlogR"] = parity.compare_logR(g["logR"], res.logR_final)
    st["events"] = parity.compare_events(g["events"], res, theta, mask)
    if name:
        parity.record(name, st)
    return st


@pytest.mark.parametrize("sigma", [0.0, 0.02])
@pytest.mark.parametrize("mode", [0, 1])
def test_c1_parity(oracle_mod, sigma, mode):
    cfg = tracegen.CONFIGS["C1"]
    x = tracegen.generate(tracegen.make_spec(cfg, sigma=sigma))
    g = _run_gpu(x, cfg.R, cfg.hazard, mode, ev_mask=3, cap=4096)
    res = _oracle(oracle_mod, x, cfg.R, cfg.hazard, mode)
    _full_check(g, res, mask=3, name=f"C1 sigma={sigma} mode={mode}")
    assert [(int(e["t"]), int(e["cp_index"])) for e in g["events"] if e["flags"] & 1] == [(600, 600)]


@pytest.mark.parametrize("R,mode,variant", [(3, "drop", 0), (3, "merge", 0), (4, "merge", 0),
                                            (5, "drop", 0), (16, "merge", 0), (16, "drop", 1),
                                            (4, "drop", 1), (2, "merge", 0), (2, "drop", 0)])
def test_bruteforce_cases_streaming(R, mode, variant):
    """T = 1 per call (streaming), posterior read after every step, vs enumeration."""
    from tests.test_oracle_bruteforce import _data
    x, pr = _data(variant)
    b = bocd.BocdBatch(1, R=R, hazard=pr["H"], kappa0=pr["k0"], alpha0=pr["a0"], mu0=pr["mu0"],
                       beta0=pr["b0"], trunc_mode=mode)
    xd = torch.from_numpy(x[None, :].copy()).cuda()
    traj = []
    for t in range(x.shape[0]):
        b.update_chunk(xd[:, t:t + 1])
        traj.append(b.read_posterior()[0].cpu().numpy()[0])
    b.close()
    ref, _ = bruteforce.posterior(x, R, pr["H"], pr["mu0"], pr["k0"], pr["a0"], pr["b0"], mode)
    for t in range(x.shape[0]):
        r = np.asarray(ref[t])
        fin = np.isfinite(r)
        assert np.all(np.abs(traj[t][fin] - r[fin]) < 1e-11), (t, traj[t], r)
        assert np.all(traj[t][~fin] < -1e300)


@pytest.mark.parametrize("mode", [0, 1])
def test_c2_subset_parity(oracle_mod, mode):
    cfg = tracegen.CONFIGS["C2"]
    spec = tracegen.make_spec(cfg)
    x = tracegen.generate(spec, 0, 24, 0, 3000)
    g = _run_gpu(x, cfg.R, cfg.hazard, mode, ev_mask=3, cap=4096)
    res = _oracle(oracle_mod, x, cfg.R, cfg.hazard, mode)
    assert not g["dropped"]
    _full_check(g, res, mask=3, name=f"C2[:24,:3000] mode={mode}")


@pytest.mark.parametrize("mode", [0, 1])
def test_c3_subset_parity(oracle_mod, mode):
    cfg = tracegen.CONFIGS["C3"]
    spec = tracegen.make_spec(cfg)
    x = tracegen.generate(spec, 0, 16, 0, 2500)
    g = _run_gpu(x, cfg.R, cfg.hazard, mode, prior_cov=cfg.prior_cov, ev_mask=3, cap=4096)
    res = _oracle(oracle_mod, x, cfg.R, cfg.hazard, mode, prior_cov=cfg.prior_cov)
    assert not g["dropped"]
    _full_check(g, res, mask=3, name=f"C3[:16,:2500] mode={mode}")


@pytest.mark.parametrize("R", [7, 100, 300, 1000])
def test_generic_R_parity(oracle_mod, R):
    cfg = tracegen.CONFIGS["C3"]
    x = tracegen.generate(tracegen.make_spec(cfg), 3, 6, 0, 1500)
    for mode in (0, 1):
        g = _run_gpu(x, R, 1 / 100, mode, prior_cov=0.3, ev_mask=3, cap=2048)
        res = _oracle(oracle_mod, x, R, 1 / 100, mode, prior_cov=0.3)
        assert not g["dropped"]
        _full_check(g, res, mask=3, name=f"C3[3:9,:1500] R={R} mode={mode}")


@pytest.mark.parametrize("R,span", [(2048, 2.5), (4096, 2.5), (2048, 10)])
def test_large_R_parity(oracle_mod, R, span):
    """The FULL kernels for R = 2048 (256 threads per series) and R = 4096 (C4: 512 threads,
    one series per CTA), past R steps so that truncation, rotation and the rebase all run;
    10 R steps: a long chain of MERGE bucket merges (its multiplicative continuation)."""
    cfg = tracegen.CONFIGS["C4"]
    x = tracegen.generate(tracegen.make_spec(cfg, n_series=64), 5, 3, 0, int(span * R))
    for mode in ((0, 1) if span < 5 else (0,)):
        g = _run_gpu(x, R, cfg.hazard, mode, prior_cov=cfg.prior_cov, ev_mask=3, cap=4096)
        res = _oracle(oracle_mod, x, R, cfg.hazard, mode, prior_cov=cfg.prior_cov)
        assert not g["dropped"]
        _full_check(g, res, mask=3, name=f"C4-recipe[5:8,:{int(span * R)}] R={R} mode={mode}")


@pytest.mark.parametrize("R,T,chunks", [(1024, 1300, [1, 255, 257, 3, 512, 1, 271]),
                                         (2048, 2600, [1, 700, 1, 2, 1300, 64, 532])])
def test_chunk_split_bit_exact(R, T, chunks):
    """Any split into calls (1-step calls run the persistent kernels) gives bit-identical
    results; R = 2048 also covers the MERGE bucket's multiplicative continuation."""
    cfg = tracegen.CONFIGS["C3"]
    x = tracegen.generate(tracegen.make_spec(cfg), 0, 8, 0, T)
    a = _run_gpu(x, R, cfg.hazard, 0, prior_cov=0.3, ev_mask=3)
    b = _run_gpu(x, R, cfg.hazard, 0, prior_cov=0.3, ev_mask=3, chunks=chunks)
    for k in ("map", "pnew", "logz", "logR", "mu", "beta"):
        assert np.array_equal(a[k], b[k], equal_nan=True), k
    assert np.array_equal(a["events"], b["events"])


def test_series_permutation_bit_exact():
    cfg = tracegen.CONFIGS["C2"]
    x = tracegen.generate(tracegen.make_spec(cfg), 0, 12, 0, 800)
    perm = np.random.default_rng(0).permutation(12)
    a = _run_gpu(x, 512, cfg.hazard, 0)
    b = _run_gpu(x[perm], 512, cfg.hazard, 0)
    for k in ("map", "pnew", "logz", "logR"):
        assert np.array_equal(a[k][perm], b[k]), k


def test_host_path_equals_device_path():
    cfg = tracegen.CONFIGS["C2"]
    x = tracegen.generate(tracegen.make_spec(cfg), 0, 10, 0, 700)
    a = _run_gpu(x, 512, cfg.hazard, 0)
    h = bocd.BocdBatch(10, R=512, hazard=cfg.hazard, prior_first_obs=True, prior_cov=0.05)
    xp = torch.from_numpy(x).pin_memory()
    m1, p1, z1 = h.update_chunk_host(xp[:, :300], outputs=True)
    m2, p2, z2 = h.update_chunk_host(xp[:, 300:], outputs=True)
    logR = h.read_posterior()[0].cpu().numpy()
    h.close()
    assert np.array_equal(np.concatenate([m1, m2], 1), a["map"])
    assert np.array_equal(np.concatenate([z1, z2], 1), a["logz"])
    assert np.array_equal(logR, a["logR"])


def test_device_tracegen_matches_numpy():
    cfg = tracegen.CONFIGS["C3"]
    spec = tracegen.make_spec(cfg, n_series=64, T=3000)
    ref = tracegen.generate(spec, 5, 40, 100, 2000)
    dt = bocd.DeviceTrace(spec, "cuda")
    out = torch.empty((40, 2000), dtype=torch.float64, device="cuda")
    dt.generate(out, 5, 100)
    np.testing.assert_allclose(out.cpu().numpy(), ref, rtol=1e-13, atol=0)


def test_nonfinite_input_is_reported():
    x = np.ones((2, 50))
    x[1, 20] = np.nan
    b = bocd.BocdBatch(2, R=64, mu0=1.0, beta0=0.01)
    b.update_chunk(torch.from_numpy(x).cuda())
    with pytest.raises(bocd.N.FalconError) as ei:
        b.changepoints()
    assert ei.value.code == bocd.N.FALCON_ENONFINITE
    with pytest.raises(bocd.N.FalconError):
        b.update_chunk(torch.from_numpy(x).cuda())
    b.close()


def test_event_overflow_warning():
    cfg = tracegen.CONFIGS["C1"]
    x = np.tile(tracegen.generate(tracegen.make_spec(cfg)), (3, 1))
    b = bocd.BocdBatch(3, R=256, hazard=cfg.hazard, prior_first_obs=True, event_mask=3,
                       event_capacity=1)
    b.update_chunk(torch.from_numpy(x).cuda())
    ev, dropped = b.changepoints()
    b.close()
    assert len(ev) == 3 and not dropped  # one PROB|MAPRESET event per series fits exactly
    b = bocd.BocdBatch(3, R=256, hazard=cfg.hazard, prior_first_obs=True, event_mask=3,
                       event_capacity=1, trunc_mode="drop")
    b.update_chunk(torch.from_numpy(x).cuda())
    ev, dropped = b.changepoints()
    b.close()
    assert len(ev) == 3 and dropped  # DROP misfires MAPRESET (reading Q6): overflow reported


def test_streaming_persistent_path_bit_exact(oracle_mod):
    """Streaming calls (T <= 64 steps, more units than co-resident CTAs) run the persistent
    kernels with TMA-prefetched state: same arithmetic as the one-unit-per-CTA kernels, so
    one-column calls equal a single long call bit for bit, and sampled series match the oracle."""
    cfg = tracegen.CONFIGS["C3"]
    S, T = 1536, 96
    spec = tracegen.make_spec(cfg, n_series=S)
    x = tracegen.generate(spec, 0, S, 0, T)
    a = _run_gpu(x, 1024, cfg.hazard, 0, prior_cov=0.3, ev_mask=1, cap=64)
    b = _run_gpu(x, 1024, cfg.hazard, 0, prior_cov=0.3, ev_mask=1, cap=64, chunks=[1] * 40 + [56])
    for k in ("map", "pnew", "logz", "logR", "mu", "beta"):
        assert np.array_equal(a[k], b[k], equal_nan=True), k
    assert np.array_equal(a["events"], b["events"])
    sample = [0, 777, 1535]
    res = _oracle(oracle_mod, x[sample], 1024, cfg.hazard, 0, prior_cov=0.3)
    st = parity.compare_steps(b["map"][sample], b["pnew"][sample], b["logz"][sample], res, 0.9)
    st["max_dlogR"] = parity.compare_logR(b["logR"][sample], res.logR_final)
    parity.record("C3[0:1536,:96] R=1024 streaming (persistent) sampled", st)
    # the on-demand-MAP (lazy) persistent kernel: no per-step outputs requested
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    h = bocd.BocdBatch(S, R=1024, hazard=cfg.hazard, prior_first_obs=True, prior_cov=0.3,
                       event_mask=1, event_capacity=64)
    for t in range(T):
        h.update_chunk(xd[:, t:t + 1])
    logR = h.read_posterior()[0].cpu().numpy()
    ev, _ = h.changepoints()
    h.close()
    assert np.array_equal(logR, a["logR"], equal_nan=True)
    assert np.array_equal(ev, a["events"])


def test_repeat_runs_bit_identical():
    """Race detector of our own (compute-sanitizer is unavailable on this pool): the same
    input twice through the resident and the persistent kernels gives identical bits."""
    cfg = tracegen.CONFIGS["C3"]
    S, T = 1536, 300
    x = tracegen.generate(tracegen.make_spec(cfg, n_series=S), 0, S, 0, T)
    for chunks in ([T], [1] * 20 + [280]):
        runs = [_run_gpu(x, 1024, cfg.hazard, 0, prior_cov=0.3, ev_mask=3, cap=256, chunks=chunks)
                for _ in range(2)]
        for k in ("map", "pnew", "logz", "logR", "mu", "beta"):
            assert np.array_equal(runs[0][k], runs[1][k], equal_nan=True), (chunks[:2], k)
        assert np.array_equal(runs[0]["events"], runs[1]["events"])


@pytest.mark.parametrize("R,mode", [(1024, 0), (1024, 1), (2048, 0), (300, 0)])
def test_lazy_map_equals_eager_map(R, mode):
    """The lazy kernel (no per-step outputs: the bench's kernel; r* = 1 at every PROB event for
    theta >= 1/2) reports exactly the PROB events of the EAGER kernel (r* reduced every step)."""
    cfg = tracegen.CONFIGS["C3"]
    x = tracegen.generate(tracegen.make_spec(cfg), 0, 64, 0, max(2 * R, 1500))
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    evs = []
    for outputs in (True, False):
        b = bocd.BocdBatch(64, R=R, hazard=cfg.hazard, prior_first_obs=True, prior_cov=0.3,
                           trunc_mode=mode, event_mask=1, event_capacity=2048)
        b.update_chunk(xd, outputs=outputs)
        ev, dropped = b.changepoints()
        b.close()
        assert not dropped
        evs.append(ev)
    assert len(evs[0]) > 0
    assert np.array_equal(evs[0], evs[1])


@pytest.mark.parametrize("R,S", [(1024, 5), (256, 13), (512, 7)])
def test_partial_cta_series_counts(oracle_mod, R, S):
    """Series counts that leave a CTA's last series groups empty (2, 8 and 4 series per CTA for
    R = 1024, 256, 512), through a long call and through 1-step (persistent-kernel) calls."""
    cfg = tracegen.CONFIGS["C3"]
    x = tracegen.generate(tracegen.make_spec(cfg), 11, S, 0, max(R + 300, 600))
    T = x.shape[1]
    a = _run_gpu(x, R, cfg.hazard, 0, prior_cov=0.3, ev_mask=1, cap=256)
    b = _run_gpu(x, R, cfg.hazard, 0, prior_cov=0.3, ev_mask=1, cap=256, chunks=[1] * 20 + [T - 20])
    for k in ("map", "pnew", "logz", "logR", "mu", "beta"):
        assert np.array_equal(a[k], b[k], equal_nan=True), k
    res = _oracle(oracle_mod, x, R, cfg.hazard, 0, prior_cov=0.3)
    _full_check(a, res, mask=1, name=f"C3[11:{11 + S},:{T}] R={R} S={S}")


@pytest.mark.parametrize("R", [256, 512, 2048, 4096, 300])
@pytest.mark.parametrize("mode", [0, 1])
def test_persistent_kernels_bit_exact(oracle_mod, R, mode):
    """Every persistent kernel (forced with falcon_bocd_set_schedule: the PREF kernels with
    TMA-prefetched state at R <= 1024, the plain persistent ones at R = 2048 / 4096 including
    the MERGE bucket's continuation, the generic-R ones) over 1-step and short calls equals
    one long one-unit-per-CTA call bit for bit, EAGER and lazy, and sampled series match the
    oracle.  S leaves the last CTA partly empty."""
    cfg = tracegen.CONFIGS["C3"]
    S = 7 if R >= 2048 else 21
    T = R + 150 if R <= 512 else 300
    x = tracegen.generate(tracegen.make_spec(cfg, n_series=64), 0, S, 0, T)
    chunks = [1] * 30 + [64, 3, 1] + [T - 98]
    a = _run_gpu(x, R, cfg.hazard, mode, prior_cov=0.3, ev_mask=3, cap=512, schedule="one_unit")
    b = _run_gpu(x, R, cfg.hazard, mode, prior_cov=0.3, ev_mask=3, cap=512, chunks=chunks,
                 schedule="persistent")
    for k in ("map", "pnew", "logz", "logR", "mu", "beta"):
        assert np.array_equal(a[k], b[k], equal_nan=True), k
    assert np.array_equal(a["events"], b["events"])
    # lazy persistent kernels (PROB only, no per-step outputs)
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    logs = []
    for sched, parts in (("one_unit", [T]), ("persistent", chunks)):
        h = bocd.BocdBatch(S, R=R, hazard=cfg.hazard, prior_first_obs=True, prior_cov=0.3, trunc_mode=mode,
                           event_mask=1, event_capacity=512)
        h.set_schedule(sched)
        t0 = 0
        for n in parts:
            h.update_chunk(xd[:, t0:t0 + n])
            t0 += n
        logs.append((h.read_posterior()[0].cpu().numpy(), h.changepoints()[0]))
        h.close()
    assert np.array_equal(logs[0][0], logs[1][0], equal_nan=True)
    assert np.array_equal(logs[0][1], logs[1][1])
    res = _oracle(oracle_mod, x[:3], R, cfg.hazard, mode, prior_cov=0.3)
    st = parity.compare_steps(b["map"][:3], b["pnew"][:3], b["logz"][:3], res, 0.9)
    st["max_dlogR"] = parity.compare_logR(b["logR"][:3], res.logR_final)
    parity.record(f"persistent R={R} mode={mode} [0:3,:{T}]", st)


@pytest.mark.parametrize("R,S", [(512, 1024), (512, 700), (1024, 400)])
@pytest.mark.parametrize("mode", [0, 1])
def test_balanced_wave_bit_exact(oracle_mod, R, S, mode):
    """A batch that fits one wave of CTAs unevenly (C2: 1,024 series of R = 512 in CTAs of 4,
    two per SM) runs as one balanced CTA per SM (capi.cu launch_update; the MINB = 1 twins of bocd_kernel.cuh):
    bit-identical to the packed one-unit launch ('one_unit_packed'), EAGER and lazy, and the
    first, a middle and the last series match the oracle."""
    cfg = tracegen.CONFIGS["C2"] if R == 512 else tracegen.CONFIGS["C3"]
    T = 300
    x = tracegen.generate(tracegen.make_spec(cfg, n_series=S), 0, S, 0, T)
    a = _run_gpu(x, R, cfg.hazard, mode, prior_cov=0.3, ev_mask=3, cap=512, schedule="auto")
    b = _run_gpu(x, R, cfg.hazard, mode, prior_cov=0.3, ev_mask=3, cap=512, schedule="one_unit_packed")
    for k in ("map", "pnew", "logz", "logR", "mu", "beta"):
        assert np.array_equal(a[k], b[k], equal_nan=True), k
    assert np.array_equal(a["events"], b["events"])
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    logs = []
    for sched in ("auto", "one_unit_packed"):  # lazy kernels (PROB only)
        h = bocd.BocdBatch(S, R=R, hazard=cfg.hazard, prior_first_obs=True, prior_cov=0.3, trunc_mode=mode,
                           event_mask=1, event_capacity=512)
        h.set_schedule(sched)
        h.update_chunk(xd)
        logs.append((h.read_posterior()[0].cpu().numpy(), h.changepoints()[0]))
        h.close()
    assert np.array_equal(logs[0][0], logs[1][0], equal_nan=True)
    assert np.array_equal(logs[0][1], logs[1][1])
    rows = [0, S // 2, S - 1]
    res = _oracle(oracle_mod, x[rows], R, cfg.hazard, mode, prior_cov=0.3)
    st = parity.compare_steps(a["map"][rows], a["pnew"][rows], a["logz"][rows], res, 0.9)
    st["max_dlogR"] = parity.compare_logR(a["logR"][rows], res.logR_final)
    parity.record(f"balanced R={R} S={S} mode={mode}", st)


@pytest.mark.parametrize("R", [1024, 4096, 1000])
@pytest.mark.parametrize("kappa0,alpha0", [(0.5, 1.5), (2.0, 0.7), (1.0, 3.0), (1.0, 0.3)])
def test_priors_and_per_series_arrays(oracle_mod, R, kappa0, alpha0):
    """kappa0, alpha0 != 1 at the BASELINE ring sizes (FULL kernels: 2 alpha_{r+1} as the exact
    integer conversion of floor(2 alpha0) + 1 + r, plus the fractional part of 2 alpha0 for
    alpha0 = 0.7 / 0.3) and at R = 1000 (the generic kernels: table-driven alpha), with
    per-series mu0 / beta0 HOST arrays passed through falcon_bocd_config (not prior_first_obs)."""
    cfg = tracegen.CONFIGS["C3"]
    S = 6
    T = R + 200 if R <= 1024 else 1200
    x = tracegen.generate(tracegen.make_spec(cfg, n_series=S), 0, S, 0, T)
    rng = np.random.default_rng(R + int(10 * alpha0))
    mu0 = x[:, 0] * rng.uniform(0.8, 1.2, S)
    beta0 = alpha0 * (rng.uniform(0.1, 0.5, S) * x[:, 0]) ** 2
    g = _run_gpu(x, R, cfg.hazard, 0, kappa0=kappa0, alpha0=alpha0, mu0=mu0, beta0=beta0, ev_mask=3, cap=2048)
    res = _oracle(oracle_mod, x, R, cfg.hazard, 0, mu0=mu0, beta0=beta0, kappa0=kappa0, alpha0=alpha0)
    assert not g["dropped"]
    _full_check(g, res, mask=3, name=f"priors R={R} kappa0={kappa0} alpha0={alpha0} per-series arrays")


@pytest.mark.parametrize("theta", [0.3, 0.5, 0.8])
def test_threshold_parity(oracle_mod, theta):
    """The PROB rule at other thresholds (P:770 fixes 0.9): theta < 1/2 runs the EAGER kernel
    (r* reduced every step), theta >= 1/2 the lazy one (r* = 1 at PROB events)."""
    cfg = tracegen.CONFIGS["C3"]
    x = tracegen.generate(tracegen.make_spec(cfg), 40, 16, 0, 1500)
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    b = bocd.BocdBatch(16, R=1024, hazard=cfg.hazard, prior_first_obs=True, prior_cov=0.3,
                       event_mask=1, event_capacity=1024, threshold=theta)
    b.update_chunk(xd)
    ev, dropped = b.changepoints()
    b.close()
    res = _oracle(oracle_mod, x, 1024, cfg.hazard, 0, prior_cov=0.3, threshold=theta)
    assert not dropped
    n = parity.compare_events(ev, res, theta, 1)
    assert n > 0
