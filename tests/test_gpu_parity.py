"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element.

Tolerance (BASELINE.json north_star): max relative error <= 1e-11 in h and u after 100 coarse
steps, normwise (reading Q26: eps_h = max|dh| / max|h|, eps_u = max|du| / max|u|), and mass /
absolute-vorticity drift <= 1e-13.  Both sides evaluate the paper's formulas in the same
canonical order without FMA contraction, so the observed difference is expected to be 0; the
tests assert the contract tolerance and record the bitwise result.
"""
import math

import numpy as np
import pytest

from inputs import configs
from oracle import diagnostics as dg
from oracle import fbrk32, lts, trisk

pytestmark = pytest.mark.gpu
TOL = 1e-11
DRIFT = 1e-13


@pytest.fixture(scope="module")
def Solver():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2405_10505_b200 import Solver
    return Solver


def phys_of(c):
    return fbrk32.Phys(g=c.g, beta=c.beta, slow=c.slow, tau_n=c.tau_n, rho0=c.rho0)


def run_oracle(c, n, M=None, fine=None):
    M = c.M if M is None else M
    fine = c.fine_mask if fine is None else fine
    lab = lts.label_regions(c.mesh, fine)
    h, u = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, M, phys_of(c), n)
    return h, u, lab


def run_gpu(Solver, c, n, M=None, fine=None):
    M = c.M if M is None else M
    fine = c.fine_mask if fine is None else fine
    s = Solver(c.mesh, fine, c.dt, M, g=c.g, beta=c.beta, rho0=c.rho0, slow=c.slow, tau_n=c.tau_n)
    s.set_state(c.h0, c.u0, 0.0)
    s.step(n)
    h, u, t = s.state()
    return s, h, u, t


def rel_err(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def assert_parity(hg, ug, ho, uo, tol=TOL):
    assert np.all(np.isfinite(hg)) and np.all(np.isfinite(ug))
    eh, eu = rel_err(hg, ho), rel_err(ug, uo)
    assert eh <= tol and eu <= tol, (eh, eu)
    return eh, eu


@pytest.mark.parametrize("which", ["config1", "shelf", "shelf_ragged"])
def test_parity_100_steps(Solver, which):
    """FB-LTS (M = 4) after 100 coarse steps: h and u within 1e-11 of the oracle (expected bitwise)."""
    c = {"config1": lambda: configs.config1(),
         "shelf": lambda: configs.small_shelf(nx=48, ny=40, dt=25.0),
         "shelf_ragged": lambda: configs.small_shelf(nx=70, ny=38, seed=11, dt=25.0)}[which]()
    n = 100
    ho, uo, lab = run_oracle(c, n)
    s, hg, ug, t = run_gpu(Solver, c, n)
    eh, eu = assert_parity(hg, ug, ho, uo)
    print(f"{which}: eps_h={eh:.3e} eps_u={eu:.3e} bitwise={np.array_equal(hg, ho) and np.array_equal(ug, uo)}")
    assert np.array_equal(hg, ho) and np.array_equal(ug, uo), "not bitwise (canonical arithmetic, --fmad=false)"
    assert t == pytest.approx(n * c.dt)
    cell, edge = s.labels()
    assert np.array_equal(cell, lab.cell) and np.array_equal(edge, lab.edge)
    m0 = dg.total_mass(c.mesh, c.h0)
    assert abs(dg.total_mass(c.mesh, hg) - m0) <= DRIFT * m0


@pytest.mark.parametrize("M", [1, 2, 3, 8])
def test_parity_other_M(Solver, M):
    """Any subcycling ratio; M = 1 reduces to FB-RK(3,2)."""
    c = configs.small_shelf(nx=48, ny=40, dt=min(5.0 * M, 30.0))      # fine nu ~ 0.5 for every M
    ho, uo, _ = run_oracle(c, 20, M=M)
    _, hg, ug, _ = run_gpu(Solver, c, 20, M=M)
    assert_parity(hg, ug, ho, uo)
    if M == 1:
        hh, uu = c.h0.copy(), c.u0.copy()
        for _ in range(20):
            hh, uu = fbrk32.fbrk32_step(c.mesh, hh, uu, c.dt, phys_of(c))
        assert_parity(hg, ug, hh, uu)


def test_parity_no_fine_cells_is_global(Solver):
    """No fine cells: the GPU runs global FB-RK(3,2) (P2; config 3's mode)."""
    c = configs.small_shelf(nx=48, ny=40, dt=4.0)
    none = np.zeros(c.mesh.nCells, bool)
    hh, uu = c.h0.copy(), c.u0.copy()
    for _ in range(30):
        hh, uu = fbrk32.fbrk32_step(c.mesh, hh, uu, c.dt, phys_of(c))
    _, hg, ug, _ = run_gpu(Solver, c, 30, fine=none)
    assert_parity(hg, ug, hh, uu)


def test_parity_all_fine(Solver):
    """Every cell fine (no coarse region): M fine FB-RK(3,2) subcycles everywhere, with the slow
    terms frozen over the whole coarse step -- so this is NOT global FB-RK(3,2) at dt/M."""
    c = configs.small_shelf(nx=40, ny=36, dt=20.0)
    allf = np.ones(c.mesh.nCells, bool)
    ho, uo, lab = run_oracle(c, 10, fine=allf)
    assert np.all(lab.cell == 8)
    _, hg, ug, _ = run_gpu(Solver, c, 10, fine=allf)
    assert_parity(hg, ug, ho, uo)
    c.slow = False                         # gravity-wave model: then it IS global FB-RK(3,2) at dt/M
    hh, uu = c.h0.copy(), c.u0.copy()
    for _ in range(10 * c.M):
        hh, uu = fbrk32.fbrk32_step(c.mesh, hh, uu, c.dt / c.M, phys_of(c))
    _, hg, ug, _ = run_gpu(Solver, c, 10, fine=allf)
    assert_parity(hg, ug, hh, uu, tol=1e-13)   # dt/(3M) vs (dt/M)/3 round differently


def test_parity_gravity_wave_model(Solver):
    """Slow terms disabled (eq. grav_wave_model)."""
    c = configs.config1()
    c.slow = False
    ho, uo, _ = run_oracle(c, 50)
    _, hg, ug, _ = run_gpu(Solver, c, 50)
    assert_parity(hg, ug, ho, uo)


def test_parity_config2_full_size(Solver):
    """BASELINE config 2 at full size (262,144 cells), 3 coarse steps, element by element."""
    c = configs.config2()
    ho, uo, _ = run_oracle(c, 3)
    _, hg, ug, _ = run_gpu(Solver, c, 3)
    assert_parity(hg, ug, ho, uo)


def test_diagnostics_match_oracle(Solver):
    """fblts_diagnostics = (mass, Gamma, min h, max nu) of the oracle (Thms 1-2, eq. cfl)."""
    c = configs.small_shelf(nx=48, ny=40, dt=25.0)
    ho, uo, lab = run_oracle(c, 10)
    s, hg, ug, _ = run_gpu(Solver, c, 10)
    d = s.diagnostics()
    ref = dg.diagnostics(c.mesh, lab, ho, uo, c.dt, c.M, c.g)
    assert d[0] == pytest.approx(ref[0], rel=1e-15)
    fscale = float(np.sum(c.mesh.areaTriangle * np.abs(c.mesh.fVertex)))
    assert abs(d[1] - ref[1]) <= 1e-15 * fscale
    assert d[2] == ref[2] and d[3] == pytest.approx(ref[3], rel=1e-15)


def test_conservation_on_gpu_long_run(Solver):
    """Theorem 1 on the GPU: mass drift <= 1e-13 over 200 coarse steps (config 1)."""
    c = configs.config1()
    s = Solver(c.mesh, c.fine_mask, c.dt, c.M)
    s.set_state(c.h0, c.u0)
    d0 = s.diagnostics()
    s.step(200)
    d1 = s.diagnostics()
    assert abs(d1[0] - d0[0]) <= DRIFT * d0[0]
    fscale = float(np.sum(c.mesh.areaTriangle * np.abs(c.mesh.fVertex)))
    assert abs(d1[1] - d0[1]) <= DRIFT * fscale


def test_comparison_can_fail(Solver):
    """Injected fault: perturbing one IF-1 value of the GPU result by 1e-9 relative must trip both
    the parity check and the conservation check (the tests can see an error of that size)."""
    c = configs.config1()
    ho, uo, lab = run_oracle(c, 10)
    _, hg, ug, _ = run_gpu(Solver, c, 10)
    i = int(np.nonzero(lab.IF1())[0][0])
    bad = hg.copy()
    bad[i] *= 1.0 + 1e-9
    with pytest.raises(AssertionError):
        assert_parity(bad, ug, ho, uo)
    m0 = dg.total_mass(c.mesh, c.h0)
    assert abs(dg.total_mass(c.mesh, bad) - m0) > DRIFT * m0


def test_deterministic(Solver):
    c = configs.small_shelf(nx=48, ny=40, dt=25.0)
    _, h1, u1, _ = run_gpu(Solver, c, 15)
    _, h2, u2, _ = run_gpu(Solver, c, 15)
    assert np.array_equal(h1, h2) and np.array_equal(u1, u2)


def test_positivity_error_is_reported(Solver):
    """A blow-up (dt far beyond the CFL limit) surfaces as FBLTS_ERR_POSITIVITY naming the kernel."""
    from paper_2405_10505_b200 import abi
    c = configs.config1(dt=2000.0)
    s = Solver(c.mesh, c.fine_mask, c.dt, c.M)
    s.set_state(c.h0, c.u0)
    s.step(100)
    with pytest.raises(abi.FbltsError) as ei:
        s.state()
    assert ei.value.code == -7 and "positivity" in str(ei.value)


def test_set_state_rejects_bad_h(Solver):
    from paper_2405_10505_b200 import abi
    c = configs.config1()
    s = Solver(c.mesh, c.fine_mask, c.dt, c.M)
    h = c.h0.copy()
    h[5] = -1.0
    h[9] = np.nan
    with pytest.raises(abi.FbltsError) as ei:
        s.set_state(h, c.u0)
    assert ei.value.code == -4 and "h[5]" in str(ei.value)         # the first offending index
    with pytest.raises(abi.FbltsError) as ei:                      # no valid state after a rejected one
        s.step(1)
    u = c.u0.copy()
    u[7] = np.inf
    with pytest.raises(abi.FbltsError) as ei:
        s.set_state(c.h0, u)
    assert ei.value.code == -4 and "u[7]" in str(ei.value)
    s.set_state(c.h0, c.u0)                                        # a good state is accepted again
    s.step(1)
    assert np.all(np.isfinite(s.state()[0]))


def test_profile_counts_launches(Solver):
    c = configs.config1()
    s = Solver(c.mesh, c.fine_mask, c.dt, c.M)
    s.set_state(c.h0, c.u0)
    prof = s.profile(2)
    assert prof["fine_s3"][1] == 2 * c.M and prof["slow_edge"][1] == 2 and prof["correct_if"][1] == 2
    assert all(ms >= 0.0 for ms, _ in prof.values())


def test_parity_sphere_100_steps(Solver):
    """Config-3 recipe (icosahedral dual, full Coriolis, global FB-RK(3,2)) at level 5, 100 steps."""
    c = configs.config3(level=5, n_steps=100)
    ho, uo, _ = run_oracle(c, 100)
    _, hg, ug, _ = run_gpu(Solver, c, 100)
    eh, eu = assert_parity(hg, ug, ho, uo)
    print(f"sphere L5: eps_h={eh:.3e} eps_u={eu:.3e}")


def test_parity_config3_full_size(Solver):
    """BASELINE config 3 at full size (655,362 cells), 3 steps, element by element."""
    c = configs.config3()
    ho, uo, _ = run_oracle(c, 3)
    _, hg, ug, _ = run_gpu(Solver, c, 3)
    assert_parity(hg, ug, ho, uo)


def test_sphere_with_fine_region(Solver):
    """FB-LTS on the sphere: a fine polar cap (M = 3) on the level-5 icosahedral dual."""
    c = configs.config3(level=5, n_steps=50)
    c.fine_mask = c.mesh.zCell > 0.6 * c.mesh.radius
    c.M = 3
    ho, uo, _ = run_oracle(c, 50)
    _, hg, ug, _ = run_gpu(Solver, c, 50)
    assert_parity(hg, ug, ho, uo)


def test_parity_config4_reduced_100_steps(Solver):
    """Config-4 recipe (variable-resolution SCVT sphere, shelf disk, M = 8, full Coriolis) at
    dx_scale = 8 (~12 k cells, maxEdges 8), 100 coarse steps element by element."""
    c = configs.config4(dx_scale=8)
    ho, uo, _ = run_oracle(c, 100)
    _, hg, ug, _ = run_gpu(Solver, c, 100)
    eh, eu = assert_parity(hg, ug, ho, uo)
    print(f"config4 (dx_scale 8): eps_h={eh:.3e} eps_u={eu:.3e}")


def test_lake_at_rest_on_gpu(Solver):
    """P6 through the GPU path: u = 0, h + z_b = const over random (integer) bathymetry, f != 0,
    slow terms on, fine region in the deep part: after 20 coarse steps the GPU state equals the
    oracle's bit for bit and moves only at roundoff (the literal FB average rounds)."""
    from inputs.hexmesh import build_periodic_hex_mesh
    m = build_periodic_hex_mesh(48, 40, 2000.0)
    rng = np.random.default_rng(6)
    H = np.round(50.0 + 3000.0 * rng.random(m.nCells))
    m.bottomDepth = H
    m.fVertex = np.full(m.nVertices, 1e-4)
    h0, u0 = H + 1.0, np.zeros(m.nEdges)
    fine = H > 1500.0
    c = configs.Case(name="lake", mesh=m, h0=h0, u0=u0, fine_mask=fine, tau_n=np.zeros(m.nEdges), M=4,
                     dt=10.0, n_steps=20)
    ho, uo, _ = run_oracle(c, 20)
    _, hg, ug, _ = run_gpu(Solver, c, 20)
    assert np.array_equal(hg, ho) and np.array_equal(ug, uo)
    assert np.max(np.abs(ug)) <= 1e-12 and np.max(np.abs(hg - h0) / h0) <= 1e-13


def test_zero_steps_is_identity(Solver):
    """step(0) enqueues nothing: the state read back is the state set (original order)."""
    c = configs.config1()
    s = Solver(c.mesh, c.fine_mask, c.dt, c.M)
    s.set_state(c.h0, c.u0, 5.0)
    s.step(0)
    h, u, t = s.state()
    assert np.array_equal(h, c.h0) and np.array_equal(u, c.u0) and t == 5.0
    s.close()


def test_unfused_and_unstaged_paths_agree(Solver, monkeypatch):
    """The staged tile kernels, the fused deep velocity + stage-1 sweep and the unstaged per-cell
    kernels are three evaluations of the same formulas: all bitwise equal (and equal to the oracle)."""
    c = configs.small_shelf(nx=64, ny=48, seed=9, dt=25.0)
    ho, uo, _ = run_oracle(c, 20)
    res = []
    for env in ({}, {"FBLTS_FUSE": "0"}, {"FBLTS_TILED": "0"}, {"FBLTS_SPLIT": "1"}, {"FBLTS_BAND_SIDE": "0"}):
        for k in ("FBLTS_FUSE", "FBLTS_TILED", "FBLTS_SPLIT", "FBLTS_BAND_SIDE"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        s, hg, ug, _ = run_gpu(Solver, c, 20)
        s.close()
        res.append((hg, ug))
    for hg, ug in res:
        assert np.array_equal(hg, ho) and np.array_equal(ug, uo)


def test_rk4_reference_scheme_matches_oracle(Solver):
    """The paper's reference scheme (classical RK4 on the unsplit system; FBLTS_SCHEME_RK4)
    through the C ABI equals the oracle's rk4_step bit for bit: config-1 mesh and state (slow terms
    on, full nonlinear PV / KE terms every stage), 50 steps at a stable RK4 step."""
    c = configs.config1()
    dt = 40.0
    phys = phys_of(c)
    h, u = c.h0.copy(), c.u0.copy()
    for _ in range(50):
        h, u = fbrk32.rk4_step(c.mesh, h, u, dt, phys)
    s = Solver(c.mesh, np.zeros(c.mesh.nCells, dtype=bool), dt, 1, g=c.g, beta=c.beta, rho0=c.rho0, slow=c.slow,
               tau_n=c.tau_n, scheme="rk4")
    s.set_state(c.h0, c.u0)
    s.step(50)
    hg, ug, _ = s.state()
    s.close()
    assert_parity(hg, ug, h, u)
    assert np.array_equal(hg, h) and np.array_equal(ug, u)


def test_rk4_with_forcing_matches_oracle(Solver):
    """RK4 with the wind-stress forcing term (config-2 recipe at reduced size)."""
    c = configs.small_shelf(nx=48, ny=40, dt=25.0)
    dt = 10.0
    phys = phys_of(c)
    h, u = c.h0.copy(), c.u0.copy()
    for _ in range(20):
        h, u = fbrk32.rk4_step(c.mesh, h, u, dt, phys)
    s = Solver(c.mesh, np.zeros(c.mesh.nCells, dtype=bool), dt, 1, g=c.g, beta=c.beta, rho0=c.rho0, slow=c.slow,
               tau_n=c.tau_n, scheme="rk4")
    s.set_state(c.h0, c.u0)
    s.step(20)
    hg, ug, _ = s.state()
    s.close()
    assert np.array_equal(hg, h) and np.array_equal(ug, u)


@pytest.mark.parametrize("which", ["config1", "shelf"])
def test_rk32_scheme_matches_oracle(Solver, which):
    """RK(3,2) of Wicker & Skamarock (FBLTS_SCHEME_RK32), the scheme FB-RK(3,2) extends,
    on the unsplit system through the C ABI equals the oracle's rk32_step bit for bit (config 1:
    slow terms, 50 steps; reduced shelf: wind-stress forcing, 30 steps)."""
    if which == "config1":
        c, dt, n = configs.config1(), 30.0, 50
    else:
        c, dt, n = configs.small_shelf(nx=48, ny=40, dt=25.0), 5.0, 30
    phys = phys_of(c)
    h, u = c.h0.copy(), c.u0.copy()
    for _ in range(n):
        h, u = fbrk32.rk32_step(c.mesh, h, u, dt, phys)
    s = Solver(c.mesh, np.zeros(c.mesh.nCells, dtype=bool), dt, 1, g=c.g, beta=c.beta, rho0=c.rho0, slow=c.slow,
               tau_n=c.tau_n, scheme="rk32")
    s.set_state(c.h0, c.u0)
    s.step(n)
    hg, ug, _ = s.state()
    s.close()
    assert_parity(hg, ug, h, u)
    assert np.array_equal(hg, h) and np.array_equal(ug, u)


@pytest.mark.parametrize("which,M", [("config1", 4), ("shelf", 2), ("shelf", 3)])
def test_slow_refresh_matches_oracle(Solver, which, M):
    """The slow-term refresh variant: S^k re-evaluated at every fine
    level on F_E through the C ABI equals the oracle's fblts_step(slow_refresh=True), 50 steps."""
    c = configs.config1() if which == "config1" else configs.small_shelf(nx=64, ny=48, seed=5, dt=25.0)
    lab = lts.label_regions(c.mesh, c.fine_mask)
    ho, uo = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, M, phys_of(c), 50, slow_refresh=True)
    s = Solver(c.mesh, c.fine_mask, c.dt, M, g=c.g, beta=c.beta, rho0=c.rho0, slow=c.slow, tau_n=c.tau_n,
               slow_refresh=True)
    s.set_state(c.h0, c.u0)
    s.step(50)
    hg, ug, _ = s.state()
    s.close()
    eh, eu = assert_parity(hg, ug, ho, uo)
    print(f"refresh {which} M={M}: eps_h={eh:.3e} eps_u={eu:.3e} bitwise={np.array_equal(hg, ho) and np.array_equal(ug, uo)}")
    assert np.array_equal(hg, ho) and np.array_equal(ug, uo), "not bitwise (canonical arithmetic, --fmad=false)"


@pytest.mark.parametrize("scheme", ["fblts", "rk4"])
def test_hurricane_terms_match_oracle(Solver, scheme):
    """Hurricane-model terms through the C ABI: SAL in the fast term,
    bottom drag and wind with the tangential reconstruction, on the synthetic hurricane shelf case
    (FB-LTS M = 4, and the RK4 reference scheme), element by element against the oracle."""
    c = configs.hurricane_case()
    phys = fbrk32.Phys(g=c.g, beta=c.beta, tau_n=c.tau_n, rho0=c.rho0, **c.hurricane)
    n = 30
    if scheme == "fblts":
        lab = lts.label_regions(c.mesh, c.fine_mask)
        ho, uo = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, c.M, phys, n)
        s = Solver(c.mesh, c.fine_mask, c.dt, c.M, g=c.g, beta=c.beta, rho0=c.rho0, tau_n=c.tau_n,
                   hurricane=c.hurricane)
    else:
        dt = 8.0
        ho, uo = c.h0.copy(), c.u0.copy()
        for _ in range(n):
            ho, uo = fbrk32.rk4_step(c.mesh, ho, uo, dt, phys)
        s = Solver(c.mesh, np.zeros(c.mesh.nCells, dtype=bool), dt, 1, g=c.g, beta=c.beta, rho0=c.rho0,
                   tau_n=c.tau_n, hurricane=c.hurricane, scheme="rk4")
    s.set_state(c.h0, c.u0)
    s.step(n)
    hg, ug, _ = s.state()
    s.close()
    eh, eu = assert_parity(hg, ug, ho, uo)
    print(f"hurricane {scheme}: eps_h={eh:.3e} eps_u={eu:.3e} bitwise={np.array_equal(hg, ho) and np.array_equal(ug, uo)}")
    assert np.array_equal(hg, ho) and np.array_equal(ug, uo), "not bitwise (canonical arithmetic, --fmad=false)"


@pytest.mark.parametrize("which,M", [("config1", 4), ("shelf", 2), ("shelf", 3), ("shelf", 1)])
def test_unsplit_matches_oracle(Solver, which, M):
    """Unsplit FB-LTS: the full Phi(U, HS) in every velocity update on
    the paper's extents, through the C ABI, against the oracle's fblts_step(split=False), 40 steps."""
    c = configs.config1() if which == "config1" else configs.small_shelf(nx=64, ny=48, seed=5,
                                                                          dt=20.0 if M > 1 else 5.0)
    lab = lts.label_regions(c.mesh, c.fine_mask)
    ho, uo = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, M, phys_of(c), 40, split=False)
    assert np.all(np.isfinite(ho))
    s = Solver(c.mesh, c.fine_mask, c.dt, M, g=c.g, beta=c.beta, rho0=c.rho0, slow=c.slow, tau_n=c.tau_n,
               unsplit=True)
    s.set_state(c.h0, c.u0)
    s.step(40)
    hg, ug, _ = s.state()
    s.close()
    eh, eu = assert_parity(hg, ug, ho, uo)
    print(f"unsplit {which} M={M}: eps_h={eh:.3e} eps_u={eu:.3e} bitwise={np.array_equal(hg, ho) and np.array_equal(ug, uo)}")
    assert np.array_equal(hg, ho) and np.array_equal(ug, uo), "not bitwise (canonical arithmetic, --fmad=false)"


@pytest.mark.parametrize("vort", [False, True])
def test_unsplit_config5_block(Solver, vort):
    """Unsplit FB-LTS on a 256 x 256 block of the config-5 recipe (M = 4; int, IF and F regions all
    thousands of cells wide): the velocity update fused into the slow edge sweep and the fine views
    restricted to the F_E slow stencil (host.cu enqueue_unsplit_step) give the oracle's
    fblts_step(split=False) bit for bit, h, u and (with the companion) eta, after 4 steps."""
    c = configs.config5(nx=256, ny=256)
    m, n = c.mesh, 4
    lab = lts.label_regions(m, c.fine_mask)
    eta0 = trisk.relative_vorticity(m, c.u0) + m.fVertex
    out = lts.run(m, lab, c.h0, c.u0, c.dt, c.M, phys_of(c), n, split=False, eta=eta0 if vort else None)
    ho, uo = out[0], out[1]
    s = Solver(m, c.fine_mask, c.dt, c.M, g=c.g, beta=c.beta, rho0=c.rho0, slow=c.slow, tau_n=c.tau_n,
               unsplit=True, vorticity=vort)
    s.set_state(c.h0, c.u0)
    if vort:
        s.set_vorticity(eta0)
    s.step(n)
    hg, ug, _ = s.state()
    eg = s.vorticity() if vort else None
    s.close()
    assert np.array_equal(hg, ho) and np.array_equal(ug, uo), "not bitwise (canonical arithmetic, --fmad=false)"
    if vort:
        assert np.array_equal(eg, out[2]), float(np.max(np.abs(eg - out[2])))


@pytest.mark.parametrize("split", [False, True])
@pytest.mark.parametrize("which,M", [("config1", 4), ("shelf", 3), ("shelf", 1)])
def test_vorticity_companion_theorem2(Solver, which, M, split):
    """Prognostic absolute vorticity companion, unsplit and split (Theorem 2; SPEC
    step_prognostic_vorticity): through the C ABI (cfg.vorticity) the eta the GPU
    advances -- the PV flux of every coarse / fine / correction velocity update, integrated per edge --
    equals the oracle's fblts_step(eta=...) bit for bit after 30 steps, and its total sum_v A_v eta_v
    is conserved to roundoff (Theorem 2); h and u stay bitwise equal too."""
    c = configs.config1() if which == "config1" else configs.small_shelf(nx=64, ny=48, seed=5,
                                                                          dt=20.0 if M > 1 else 5.0)
    m = c.mesh
    n = 30
    lab = lts.label_regions(m, c.fine_mask)
    eta0 = trisk.relative_vorticity(m, c.u0) + m.fVertex
    ho, uo, eo = lts.run(m, lab, c.h0, c.u0, c.dt, M, phys_of(c), n, split=split, eta=eta0)
    s = Solver(m, c.fine_mask, c.dt, M, g=c.g, beta=c.beta, rho0=c.rho0, slow=c.slow, tau_n=c.tau_n,
               unsplit=not split, vorticity=True)
    s.set_state(c.h0, c.u0)
    s.set_vorticity(eta0)
    s.step(n)
    hg, ug, _ = s.state()
    eg = s.vorticity()
    s.close()
    assert np.array_equal(hg, ho) and np.array_equal(ug, uo)
    assert np.array_equal(eg, eo), float(np.max(np.abs(eg - eo)))
    scale = float(np.sum(m.areaTriangle * np.abs(eta0)))
    drift = abs(float(np.sum(m.areaTriangle * eg)) - float(np.sum(m.areaTriangle * eta0))) / scale
    print(f"vorticity companion {which} M={M} split={split}: bitwise, Theorem-2 drift {drift:.2e}")
    assert drift <= 1e-13
    assert np.max(np.abs(eg - eta0)) > 0.0


@pytest.mark.parametrize("M", [1, 2, 4])
def test_fused_subcycle_matches_oracle(Solver, monkeypatch, M):
    """The fused fine subcycle (one CTA advances a tile of F\\F^5 -- or of F\\F^2 with
    FBLTS_SUB_LEVEL=2 -- through velocity stage 3 of subcycle k-1 and thickness stages 1-3 of k,
    recomputing the stage values on its rings; opt-in, FBLTS_SUB=1) evaluates the same formulas as the
    per-stage sweeps: bitwise equal to them (the default) and to the oracle, on a 256 x 256 block of
    the config-5 recipe."""
    c = configs.config5(nx=256, ny=256)
    c.dt = c.dt * M / c.M                  # the same fine step dt/M for every M (stable)
    n = 3
    ho, uo, _ = run_oracle(c, n, M=M)
    res = []
    for env in ({"FBLTS_SUB": "1"}, {"FBLTS_SUB": "1", "FBLTS_SUB_LEVEL": "2"}, {}):
        for k in ("FBLTS_SUB", "FBLTS_SUB_LEVEL"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        s, hg, ug, _ = run_gpu(Solver, c, n, M=M)
        cnt = s.counts()
        assert (cnt["sub_tiles"] > 0) == ("FBLTS_SUB" in env), cnt
        s.close()
        res.append((hg, ug))
    for hg, ug in res:
        assert_parity(hg, ug, ho, uo)
        assert np.array_equal(hg, ho) and np.array_equal(ug, uo)


@pytest.mark.parametrize("case", ["config1", "shelf_ragged", "rk4", "unsplit"])
def test_energy_pv_matches_oracle(Solver, case):
    """Energy-conserving PV flux (oracle trisk.pv_flux_energy): FB-LTS, classical RK4
    and unsplit FB-LTS with the variant, element by element against the oracle (expected bitwise)."""
    import dataclasses
    c = configs.config1() if case == "config1" else configs.small_shelf(nx=70, ny=38, seed=11, dt=25.0)
    M = 3 if case == "shelf_ragged" else c.M
    phys = dataclasses.replace(phys_of(c), pv="energy")
    lab = lts.label_regions(c.mesh, c.fine_mask)
    n = 30
    if case == "rk4":
        dt = 5.0
        ho, uo = c.h0.copy(), c.u0.copy()
        for _ in range(n):
            ho, uo = fbrk32.rk4_step(c.mesh, ho, uo, dt, phys)
        s = Solver(c.mesh, c.fine_mask, dt, 1, g=c.g, beta=c.beta, rho0=c.rho0, tau_n=c.tau_n, scheme="rk4",
                   pv="energy")
    else:
        unsplit = case == "unsplit"
        ho, uo = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, M, phys, n, split=not unsplit)
        s = Solver(c.mesh, c.fine_mask, c.dt, M, g=c.g, beta=c.beta, rho0=c.rho0, tau_n=c.tau_n,
                   unsplit=unsplit, pv="energy")
    s.set_state(c.h0, c.u0)
    s.step(n)
    hg, ug, _ = s.state()
    assert_parity(hg, ug, ho, uo)
    assert np.array_equal(hg, ho) and np.array_equal(ug, uo)
    hc, uc, _ = run_oracle(c, n, M=M) if case != "rk4" else (None, None, None)
    if uc is not None:
        assert not np.array_equal(uc, ug)              # the variant is active


def test_diagnostics_async_match_sync(Solver):
    """fblts_diagnostics_async gives, bit for bit, what fblts_diagnostics gives for the state at the
    call, even when later steps (enqueued before any sync) overwrite that state's buffers."""
    c = configs.config1()
    s = Solver(c.mesh, c.fine_mask, c.dt, c.M, g=c.g, beta=c.beta, rho0=c.rho0, tau_n=c.tau_n)
    s.set_state(c.h0, c.u0)
    want = [s.diagnostics()]
    for _ in range(6):
        s.step(1)
        want.append(s.diagnostics())
    s.set_state(c.h0, c.u0)
    got = [s.diagnostics_async()]
    for _ in range(6):
        s.step(1)
        got.append(s.diagnostics_async())
    s.step(3)                                        # overwrites both state buffers before any sync
    h, _, _ = s.state()
    for g_, w in zip(got, want):
        assert np.array_equal(g_, w), (g_, w)
    assert np.all(np.isfinite(h))


def test_diagnostics_mass_async_match_sync(Solver):
    """fblts_diagnostics_mass_async (the bench's per-step monitor) gives, bit for bit, the (mass, min h)
    fblts_diagnostics_mass gives for the state at the call, with later steps enqueued before any sync."""
    c = configs.small_shelf(nx=48, ny=40, dt=25.0)
    s = Solver(c.mesh, c.fine_mask, c.dt, c.M, g=c.g, beta=c.beta, rho0=c.rho0, tau_n=c.tau_n)
    s.set_state(c.h0, c.u0)
    want = [s.diagnostics_mass()]
    for _ in range(8):
        s.step(1)
        want.append(s.diagnostics_mass())
    s.set_state(c.h0, c.u0)
    got = [s.diagnostics_mass_async()]
    for _ in range(8):
        s.step(1)
        got.append(s.diagnostics_mass_async())
    s.step(3)
    s.sync()
    for g_, w in zip(got, want):
        assert np.array_equal(g_, w), (g_, w)
    s.close()


def test_diagnostics_mass_is_cell_part(Solver):
    """fblts_diagnostics_mass = (mass, min h) of fblts_diagnostics, bit for bit, and the oracle's."""
    c = configs.config1()
    s = Solver(c.mesh, c.fine_mask, c.dt, c.M, g=c.g, beta=c.beta, rho0=c.rho0, tau_n=c.tau_n)
    s.set_state(c.h0, c.u0)
    for _ in range(4):
        s.step(1)
        d, dm = s.diagnostics(), s.diagnostics_mass()
        assert dm[0] == d[0] and dm[1] == d[2]
    h, _, _ = s.state()
    m0 = dg.total_mass(c.mesh, h)
    assert abs(dm[0] - m0) <= 1e-15 * m0 and dm[1] == np.min(h)


def test_fused_subcycle_on_scvt_sphere(Solver, monkeypatch):
    """The opt-in fused subcycle on the variable-resolution SCVT sphere (config-4 recipe at
    dx_scale 4: pentagons to octagons, row stride G = 8, M = 8): bitwise equal to the oracle."""
    c = configs.config4(dx_scale=4)
    n = 5
    ho, uo, _ = run_oracle(c, n)
    monkeypatch.setenv("FBLTS_SUB", "1")
    s, hg, ug, _ = run_gpu(Solver, c, n)
    cnt = s.counts()
    s.close()
    if cnt["sub_tiles"] == 0:
        pytest.skip(f"no subcycle tiles on this mesh ({cnt['cells_by_region']})")
    assert_parity(hg, ug, ho, uo)
    assert np.array_equal(hg, ho) and np.array_equal(ug, uo)


def test_pv_volume_integral_on_gpu(Solver):
    """The PV volume integral sum_v A_v h_v q_v (Remark rmk:volume_conservation_pv)
    computed on the device (fblts_diagnostics_pv) equals the oracle's total_pv_volume to 1e-14 relative
    on a stepped state, and is conserved over 50 FB-LTS steps to 1e-13 of sum_v A_v |f_v| (it equals
    Gamma up to rounding, Theorem 2)."""
    c = configs.small_shelf(nx=48, ny=40, dt=25.0)
    s = Solver(c.mesh, c.fine_mask, c.dt, c.M, g=c.g, beta=c.beta, rho0=c.rho0, slow=c.slow, tau_n=c.tau_n)
    s.set_state(c.h0, c.u0)
    p0 = s.pv_volume()
    s.step(50)
    h, u, _ = s.state()
    p1 = s.pv_volume()
    s.close()
    ref = dg.total_pv_volume(c.mesh, h, u)
    scale = float(np.sum(c.mesh.areaTriangle * np.abs(c.mesh.fVertex)))
    assert abs(p1 - ref) <= 1e-14 * scale
    assert abs(p0 - dg.total_pv_volume(c.mesh, c.h0, c.u0)) <= 1e-14 * scale
    assert abs(p1 - p0) <= 1e-13 * scale
