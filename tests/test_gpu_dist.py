"""Partitioned (multi-rank) path on ONE GPU through the loopback group (fblts_step_group): the
dual-set partition, local numbering, halo lists, pack/unpack and per-rank diagnostics.  Results
must be bit-identical to the single-rank run (and hence to the oracle) for any rank count
("results bitwise identical for 1/2/4/8 GPUs")."""
import numpy as np
import pytest

from inputs import configs
from oracle import fbrk32, lts

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2405_10505_b200 import Solver, SolverGroup
    return Solver, SolverGroup


def single(Solver, c, n):
    s = Solver(c.mesh, c.fine_mask, c.dt, c.M, g=c.g, beta=c.beta, rho0=c.rho0, slow=c.slow, tau_n=c.tau_n)
    s.set_state(c.h0, c.u0)
    s.step(n)
    h, u, _ = s.state()
    d = s.diagnostics()
    s.close()
    return h, u, d


@pytest.mark.parametrize("nranks", [2, 3, 4, 8])
@pytest.mark.parametrize("which", ["config1", "shelf"])
def test_group_bitwise_equals_single_rank(mods, which, nranks):
    Solver, SolverGroup = mods
    c = configs.config1() if which == "config1" else configs.small_shelf(nx=64, ny=48, seed=5, dt=25.0)
    n = 20
    h1, u1, d1 = single(Solver, c, n)
    g = SolverGroup(c.mesh, c.fine_mask, c.dt, c.M, nranks, g=c.g, beta=c.beta, rho0=c.rho0, slow=c.slow,
                    tau_n=c.tau_n)
    g.set_state(c.h0, c.u0)
    g.step(n)
    h, u, t = g.state()
    assert np.array_equal(h, h1), np.nanmax(np.abs(h - h1))
    assert np.array_equal(u, u1), np.nanmax(np.abs(u - u1))
    d = g.diagnostics()
    assert d[0] == pytest.approx(d1[0], rel=1e-15) and d[2] == d1[2] and d[3] == d1[3]
    owned = sum(x["owned_cells"] for x in g.counts())
    assert owned == c.mesh.nCells
    g.close()


def test_group_matches_oracle(mods):
    _, SolverGroup = mods
    c = configs.small_shelf(nx=64, ny=48, seed=5, dt=25.0)
    lab = lts.label_regions(c.mesh, c.fine_mask)
    phys = fbrk32.Phys(g=c.g, beta=c.beta, slow=c.slow, tau_n=c.tau_n, rho0=c.rho0)
    ho, uo = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, c.M, phys, 30)
    g = SolverGroup(c.mesh, c.fine_mask, c.dt, c.M, 4, tau_n=c.tau_n)
    g.set_state(c.h0, c.u0)
    g.step(30)
    h, u, _ = g.state()
    assert np.array_equal(h, ho) and np.array_equal(u, uo)
    g.close()


def test_group_on_sphere(mods):
    """Partitioned run on the sphere (3-D Morton SFC), with a fine polar cap: bitwise = single rank."""
    Solver, SolverGroup = mods
    c = configs.config3(level=5, n_steps=20)
    c.fine_mask = c.mesh.zCell > 0.6 * c.mesh.radius
    c.M = 3
    h1, u1, _ = single(Solver, c, 20)
    g = SolverGroup(c.mesh, c.fine_mask, c.dt, c.M, 4)
    g.set_state(c.h0, c.u0)
    g.step(20)
    h, u, _ = g.state()
    assert np.array_equal(h, h1) and np.array_equal(u, u1)
    g.close()


@pytest.mark.parametrize("nranks", [2, 3, 4])
def test_weak_pieces_reproduce_the_block(mods, nranks):
    """Weak scaling's distributed set-up (reading Q25; fblts_set_partition): nranks ranks each build
    ONLY their piece of the config-5 recipe stacked nranks times in y (inputs.configs.config5_weak_piece)
    and step together through the loopback group.  The whole mesh is periodic with the block, so every
    rank's owned rows must equal the one-rank run of the block itself bit for bit -- the weak-scaled
    multi-GPU path computes exactly config 5's arithmetic on every GPU."""
    Solver, SolverGroup = mods
    nx = ny = 128
    n = 6
    blk = configs.config5_weak_piece(0, 1, nx=nx, ny=ny).case
    h1, u1, _ = single(Solver, blk, n)
    pieces = [configs.config5_weak_piece(r, nranks, nx=nx, ny=ny) for r in range(nranks)]
    c0 = pieces[0].case
    g = SolverGroup.from_pieces(pieces, c0.dt, c0.M, g=c0.g, beta=c0.beta, rho0=c0.rho0, slow=c0.slow,
                                tau_n=c0.tau_n)
    for s, p in zip(g.solvers, pieces):
        s.set_state(p.case.h0, p.case.u0)
    g.step(n)
    for s, p in zip(g.solvers, pieces):
        h = np.full(p.case.mesh.nCells, np.nan)
        u = np.full(p.case.mesh.nEdges, np.nan)
        s.state(h, u)
        assert np.array_equal(h[p.own], h1[p.block_cell[p.own]])
        # edges 3c+k belong to cell c in the lattice numbering: the owned cells' edges
        e = (3 * p.own[:, None] + np.arange(3)[None, :]).ravel()
        eb = (3 * p.block_cell[p.own][:, None] + np.arange(3)[None, :]).ravel()
        assert np.array_equal(u[e], u1[eb])
    d = g.diagnostics()
    assert np.isfinite(d).all()
    g.close()
