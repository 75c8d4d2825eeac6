"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/fblts.h declares,
and its host logic (mesh validation, LTS labelling) matches the oracle.  No compute calls."""
import os
import re

import numpy as np
import pytest

from inputs.configs import config1, small_shelf
from inputs.hexmesh import build_periodic_hex_mesh
from oracle import lts

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def abi():
    from paper_2405_10505_b200 import build
    build.build()
    import paper_2405_10505_b200._abi as a
    return a


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "fblts.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fblts_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(abi):
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(abi._lib, s), s
    assert sorted(abi.EXPORTED) == syms


def test_kernel_names(abi):
    names = [abi.fblts_kernel_name(k) for k in range(abi.NUM_KERNELS)]
    assert names[0] == "slow_pre" and names[-1] == "fine_sub" and len(set(names)) == abi.NUM_KERNELS


@pytest.mark.parametrize("which", ["cfg1", "shelf", "shelf_big"])
def test_library_labels_match_oracle(abi, which):
    """a0: the library's region labels (host C++) equal the oracle's, code for code."""
    c = {"cfg1": lambda: config1(), "shelf": lambda: small_shelf(nx=40, ny=36),
         "shelf_big": lambda: small_shelf(nx=96, ny=80, seed=3)}[which]()
    ctx = abi.fblts_create(c.dt, c.M)
    try:
        abi.fblts_upload_mesh(ctx, c.mesh)
        abi.fblts_set_regions(ctx, c.fine_mask)
        cell, edge = abi.fblts_get_labels(ctx, c.mesh.nCells, c.mesh.nEdges)
        lab = lts.label_regions(c.mesh, c.fine_mask)
        assert np.array_equal(cell, lab.cell) and np.array_equal(edge, lab.edge)
        cnt = abi.fblts_get_counts(ctx)
        assert list(cnt[:3]) == [c.mesh.nCells, c.mesh.nEdges, c.mesh.nVertices]
        assert list(cnt[3:12]) == list(np.bincount(lab.cell, minlength=9))
        assert list(cnt[12:21]) == list(np.bincount(lab.edge, minlength=9))
        assert abi.fblts_workspace_size(ctx) > 8 * (c.mesh.nCells + c.mesh.nEdges)
    finally:
        abi.fblts_destroy(ctx)


def test_mesh_validation_names_field_and_index(abi):
    """a broken mesh is rejected with a message naming the field and index."""
    m = build_periodic_hex_mesh(8, 6, 1000.0)
    m.cellsOnEdge = m.cellsOnEdge.copy()
    m.cellsOnEdge[7] = [m.cellsOnEdge[7, 0], m.cellsOnEdge[7, 0]]
    ctx = abi.fblts_create(10.0, 2)
    try:
        with pytest.raises(abi.FbltsError) as ei:
            abi.fblts_upload_mesh(ctx, m)
        assert ei.value.code == -2 and "cellsOnEdge[7]" in str(ei.value)
    finally:
        abi.fblts_destroy(ctx)
    m = build_periodic_hex_mesh(8, 6, 1000.0)
    m.edgesOnCell = m.edgesOnCell.copy()
    m.edgesOnCell[3, 2] = m.edgesOnCell[20, 0]
    ctx = abi.fblts_create(10.0, 2)
    try:
        with pytest.raises(abi.FbltsError) as ei:
            abi.fblts_upload_mesh(ctx, m)
        assert ei.value.code == -2 and "edgesOnCell[3][2]" in str(ei.value)
    finally:
        abi.fblts_destroy(ctx)


def test_call_order_and_args(abi):
    """Out-of-order calls return FBLTS_ERR_ORDER; bad configs FBLTS_ERR_INVALID_ARG."""
    with pytest.raises(abi.FbltsError):
        abi.fblts_create(-1.0, 4)
    with pytest.raises(abi.FbltsError):
        abi.fblts_create(10.0, 0)
    ctx = abi.fblts_create(10.0, 2)
    try:
        with pytest.raises(abi.FbltsError) as ei:
            abi.fblts_set_regions(ctx, np.zeros(16, np.uint8))
        assert ei.value.code == -8
        with pytest.raises(abi.FbltsError) as ei:
            abi.fblts_step(ctx, 1)
        assert ei.value.code == -8
    finally:
        abi.fblts_destroy(ctx)


def test_rk4_scheme_is_single_rank(abi):
    """FBLTS_SCHEME_RK4 is the one-rank reference scheme: asking for it with two ranks is rejected."""
    with pytest.raises(abi.FbltsError) as ei:
        abi.fblts_create(10.0, 1, scheme="rk4", nranks=2, rank=0)
    assert ei.value.code == -1


def test_subcycle_tiles_host_logic(abi, monkeypatch):
    """Host side of the opt-in fused subcycle (FBLTS_SUB=1), no device: on a 128 x 128 block of the
    config-5 recipe the subcycle tiles cover exactly the cells of F \\ F^5 (region code 8), their
    ring lists and edge lists are non-empty, and the footprint fits the 227 KB of shared memory;
    without the flag there are none."""
    from inputs import configs
    c = configs.config5(nx=128, ny=128)
    for flag in ("1", None):
        if flag:
            monkeypatch.setenv("FBLTS_SUB", flag)
        else:
            monkeypatch.delenv("FBLTS_SUB", raising=False)
        ctx = abi.fblts_create(c.dt, c.M)
        try:
            abi.fblts_upload_mesh(ctx, c.mesh)
            abi.fblts_set_regions(ctx, c.fine_mask)
            o = abi.fblts_get_counts(ctx)
        finally:
            abi.fblts_destroy(ctx)
        n_tiles, n_ring, n_fedge, smem = (int(x) for x in o[28:32])
        if flag:
            deep = int(o[3 + 8])
            assert deep > 0 and n_tiles >= deep // 256 and n_ring > 0 and n_fedge > 0
            assert 0 < smem <= 227 * 1024
        else:
            assert n_tiles == 0 and smem == 0
