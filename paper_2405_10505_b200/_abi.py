"""ctypes binding of libfblts.so (include/fblts.h): argument marshalling only.

Every function here has the C name of the entry point it wraps.  No arithmetic of
the method happens in Python: each call converts numpy arrays / torch tensors to
pointers and forwards them.  If the shared library is missing this module raises
ImportError -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libfblts.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2405_10505_b200.build` "
                      "(or __graft_entry__.build()); there is no CPU fallback")
_lib = C.CDLL(LIB_PATH)

FBLTS_OK = 0
ERRORS = {-1: "INVALID_ARG", -2: "MESH", -3: "LABELS", -4: "STATE", -5: "CUDA", -6: "NCCL", -7: "POSITIVITY",
          -8: "ORDER"}
NUM_KERNELS = 15

_i32p = C.POINTER(C.c_int32)
_f64p = C.POINTER(C.c_double)


class fblts_mesh(C.Structure):
    _fields_ = [("nCells", C.c_int32), ("nEdges", C.c_int32), ("nVertices", C.c_int32),
                ("maxEdges", C.c_int32), ("maxEdges2", C.c_int32),
                ("nEdgesOnCell", _i32p), ("edgesOnCell", _i32p), ("cellsOnEdge", _i32p),
                ("verticesOnEdge", _i32p), ("nEdgesOnEdge", _i32p), ("edgesOnEdge", _i32p),
                ("weightsOnEdge", _f64p), ("edgesOnVertex", _i32p), ("cellsOnVertex", _i32p),
                ("kiteAreasOnVertex", _f64p), ("areaCell", _f64p), ("areaTriangle", _f64p),
                ("dvEdge", _f64p), ("dcEdge", _f64p), ("fVertex", _f64p), ("bottomDepth", _f64p),
                ("xCell", _f64p), ("yCell", _f64p), ("zCell", _f64p)]


class fblts_config(C.Structure):
    _fields_ = [("dt", C.c_double), ("g", C.c_double), ("beta", C.c_double * 3), ("rho0", C.c_double),
                ("M", C.c_int32), ("r", C.c_int32), ("slow", C.c_int32), ("device", C.c_int32),
                ("stream", C.c_void_p), ("rank", C.c_int32), ("nranks", C.c_int32), ("nccl_id", C.c_void_p),
                ("scheme", C.c_int32), ("slow_refresh", C.c_int32), ("sal_beta", C.c_double),
                ("unsplit", C.c_int32), ("pv_energy", C.c_int32), ("vorticity", C.c_int32)]

SCHEMES = {"fblts": 0, "rk4": 1, "rk32": 2}


class FbltsError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"FBLTS_ERR_{ERRORS.get(code, code)} ({code}): {msg}")
        self.code = code


def _sig(name, res, *args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_vp = C.c_void_p
_lib_create = _sig("fblts_create", C.c_int, C.POINTER(_vp), C.POINTER(fblts_config))
_lib_upload = _sig("fblts_upload_mesh", C.c_int, _vp, C.POINTER(fblts_mesh))
_lib_regions = _sig("fblts_set_regions", C.c_int, _vp, C.POINTER(C.c_uint8))
_lib_labels = _sig("fblts_get_labels", C.c_int, _vp, C.POINTER(C.c_int8), C.POINTER(C.c_int8))
_lib_counts = _sig("fblts_get_counts", C.c_int, _vp, C.POINTER(C.c_int64))
_lib_wsize = _sig("fblts_workspace_size", C.c_int, _vp, C.POINTER(C.c_size_t))
_lib_bind = _sig("fblts_bind_workspace", C.c_int, _vp, _vp, C.c_size_t)
_lib_forcing = _sig("fblts_set_forcing", C.c_int, _vp, _f64p)
_lib_hurricane = _sig("fblts_set_hurricane", C.c_int, _vp, _f64p, _f64p, C.c_double, C.c_double)
_lib_set_state = _sig("fblts_set_state", C.c_int, _vp, _f64p, _f64p, C.c_double)
_lib_step = _sig("fblts_step", C.c_int, _vp, C.c_int32)
_lib_sync = _sig("fblts_sync", C.c_int, _vp)
_lib_get_state = _sig("fblts_get_state", C.c_int, _vp, _f64p, _f64p, C.POINTER(C.c_double))
_lib_diag = _sig("fblts_diagnostics", C.c_int, _vp, _f64p)
_lib_diag_async = _sig("fblts_diagnostics_async", C.c_int, _vp, _f64p)
_lib_diag_mass = _sig("fblts_diagnostics_mass", C.c_int, _vp, _f64p)
_lib_diag_mass_async = _sig("fblts_diagnostics_mass_async", C.c_int, _vp, _f64p)
_lib_profile = _sig("fblts_profile", C.c_int, _vp, C.c_int32, _f64p, C.POINTER(C.c_int64))
_lib_kname = _sig("fblts_kernel_name", C.c_char_p, C.c_int32)
_lib_last_error = _sig("fblts_last_error", C.c_char_p, _vp)
_lib_build_info = _sig("fblts_build_info", C.c_char_p)
_lib_set_part = _sig("fblts_set_partition", C.c_int, _vp, C.POINTER(C.c_int32), C.POINTER(C.c_int64))
_lib_diag_pv = _sig("fblts_diagnostics_pv", C.c_int, _vp, _f64p)
_lib_set_vort = _sig("fblts_set_vorticity", C.c_int, _vp, _f64p)
_lib_get_vort = _sig("fblts_get_vorticity", C.c_int, _vp, _f64p)
_lib_destroy = _sig("fblts_destroy", None, _vp)
_i64p = C.POINTER(C.c_int64)
_lib_halo = _sig("fblts_get_halo", C.c_int, _vp, C.c_int32, C.c_int32, _i64p, _i64p, _i64p, _i64p)
_lib_uid = _sig("fblts_nccl_unique_id", C.c_int, C.c_void_p)
_lib_step_group = _sig("fblts_step_group", C.c_int, C.POINTER(_vp), C.c_int32, C.c_int32)
_lib_diag_group = _sig("fblts_diagnostics_group", C.c_int, C.POINTER(_vp), C.c_int32, _f64p)

EXPORTED = ["fblts_create", "fblts_upload_mesh", "fblts_set_regions", "fblts_get_labels", "fblts_get_counts",
            "fblts_get_halo", "fblts_nccl_unique_id", "fblts_workspace_size", "fblts_bind_workspace",
            "fblts_set_forcing", "fblts_set_hurricane", "fblts_set_state", "fblts_step", "fblts_step_group", "fblts_diagnostics_group",
            "fblts_sync", "fblts_get_state", "fblts_diagnostics", "fblts_diagnostics_async", "fblts_diagnostics_mass",
            "fblts_profile",
            "fblts_kernel_name", "fblts_build_info", "fblts_set_vorticity", "fblts_get_vorticity", "fblts_diagnostics_pv", "fblts_set_partition", "fblts_diagnostics_mass_async",
            "fblts_last_error", "fblts_destroy"]


def _check(ctx, rc):
    if rc != FBLTS_OK:
        msg = _lib_last_error(ctx).decode() if ctx else ""
        raise FbltsError(rc, msg)


def _ptr(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def _arr(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# ------------------------------------------------------------------ entry points
def fblts_create(dt, M, g=9.81, beta=(0.531, 0.531, 0.313), rho0=1000.0, r=2, slow=True, device=0,
                 stream=None, rank=0, nranks=1, nccl_id=None, scheme="fblts", slow_refresh=False, sal=0.0, unsplit=False,
                 pv="centered", vorticity=False):
    """nccl_id: 128 bytes from fblts_nccl_unique_id() on rank 0 (None: single rank or loopback group)."""
    idbuf = (C.c_uint8 * 128).from_buffer_copy(nccl_id) if nccl_id is not None else None
    cfg = fblts_config(dt=float(dt), g=float(g), beta=(C.c_double * 3)(*beta), rho0=float(rho0), M=int(M),
                       r=int(r), slow=1 if slow else 0, device=int(device), stream=stream, rank=int(rank),
                       nranks=int(nranks), nccl_id=C.cast(idbuf, C.c_void_p) if idbuf is not None else None,
                       scheme=SCHEMES[scheme], slow_refresh=1 if slow_refresh else 0, sal_beta=float(sal),
                       unsplit=1 if unsplit else 0, pv_energy={"centered": 0, "energy": 1}[pv],
                       vorticity=1 if vorticity else 0)
    ctx = _vp()
    rc = _lib_create(C.byref(ctx), C.byref(cfg))
    if rc != FBLTS_OK:
        raise FbltsError(rc, "fblts_create failed (check dt, M, r, g, rho0, rank/nranks, device)")
    return ctx


def fblts_upload_mesh(ctx, mesh):
    """mesh: any object with the MPAS field names of inputs.trisk_mesh.Mesh."""
    keep = {}
    i32 = lambda k: keep.setdefault(k, _arr(getattr(mesh, k), np.int32))
    f64 = lambda k: keep.setdefault(k, _arr(getattr(mesh, k), np.float64))
    m = fblts_mesh(nCells=mesh.nCells, nEdges=mesh.nEdges, nVertices=mesh.nVertices, maxEdges=mesh.maxEdges,
                   maxEdges2=mesh.maxEdges2)
    for k in ("nEdgesOnCell", "edgesOnCell", "cellsOnEdge", "verticesOnEdge", "nEdgesOnEdge", "edgesOnEdge",
              "edgesOnVertex", "cellsOnVertex"):
        setattr(m, k, _ptr(i32(k), C.c_int32))
    for k in ("weightsOnEdge", "kiteAreasOnVertex", "areaCell", "areaTriangle", "dvEdge", "dcEdge", "fVertex",
              "bottomDepth", "xCell", "yCell", "zCell"):
        setattr(m, k, _ptr(f64(k), C.c_double))
    _check(ctx, _lib_upload(ctx, C.byref(m)))
    _MESH_SIZES[_key(ctx)] = (int(mesh.nCells), int(mesh.nEdges))


def fblts_set_regions(ctx, fine_mask):
    a = _arr(fine_mask, np.uint8)
    _check_len(a, _sizes(ctx)[0], "fine_mask")
    _check(ctx, _lib_regions(ctx, _ptr(a, C.c_uint8)))


def fblts_set_partition(ctx, owner, cell_gid):
    """Distributed set-up: the uploaded mesh is this rank's piece; owner / cell_gid per piece cell."""
    o, g = _arr(owner, np.int32), _arr(cell_gid, np.int64)
    nC = _sizes(ctx)[0]
    _check_len(o, nC, "owner")
    _check_len(g, nC, "cell_gid")
    _check(ctx, _lib_set_part(ctx, _ptr(o, C.c_int32), _ptr(g, C.c_int64)))


def fblts_get_labels(ctx, nCells, nEdges):
    cell = np.empty(nCells, np.int8)
    edge = np.empty(nEdges, np.int8)
    _check(ctx, _lib_labels(ctx, _ptr(cell, C.c_int8), _ptr(edge, C.c_int8)))
    return cell, edge


def fblts_get_counts(ctx):
    out = np.zeros(32, np.int64)
    _check(ctx, _lib_counts(ctx, _ptr(out, C.c_int64)))
    return out


def fblts_get_halo(ctx, which, peer):
    """(send global ids, recv global ids) of halo exchange `which` (0 ring-1 cells, 1 rings 1-2
    cells, 2 remote-owned edges) with `peer`."""
    ns, nr = C.c_int64(), C.c_int64()
    _check(ctx, _lib_halo(ctx, int(which), int(peer), C.byref(ns), C.byref(nr), None, None))
    snd = np.zeros(ns.value, np.int64)
    rcv = np.zeros(nr.value, np.int64)
    _check(ctx, _lib_halo(ctx, int(which), int(peer), C.byref(ns), C.byref(nr), _ptr(snd, C.c_int64),
                          _ptr(rcv, C.c_int64)))
    return snd, rcv


def fblts_nccl_unique_id():
    buf = (C.c_uint8 * 128)()
    rc = _lib_uid(C.cast(buf, C.c_void_p))
    if rc != FBLTS_OK:
        raise FbltsError(rc, "ncclGetUniqueId failed")
    return bytes(buf)


def fblts_step_group(ctxs, n_coarse):
    arr = (_vp * len(ctxs))(*[c.value if isinstance(c, _vp) else c for c in ctxs])
    _check(ctxs[0], _lib_step_group(arr, len(ctxs), int(n_coarse)))


def fblts_diagnostics_group(ctxs):
    arr = (_vp * len(ctxs))(*[c.value if isinstance(c, _vp) else c for c in ctxs])
    out = np.zeros(4)
    _check(ctxs[0], _lib_diag_group(arr, len(ctxs), _ptr(out, C.c_double)))
    return out


def fblts_workspace_size(ctx):
    n = C.c_size_t()
    _check(ctx, _lib_wsize(ctx, C.byref(n)))
    return n.value


def fblts_bind_workspace(ctx, device_ptr, nbytes):
    _check(ctx, _lib_bind(ctx, _vp(device_ptr), nbytes))


def fblts_set_forcing(ctx, tau_n):
    if tau_n is None:
        _check(ctx, _lib_forcing(ctx, None))
    else:
        a = _arr(tau_n, np.float64)
        _check_len(a, _sizes(ctx)[1], "tau_n")
        _check(ctx, _lib_forcing(ctx, _ptr(a, C.c_double)))


def fblts_set_hurricane(ctx, uw_n, uw_t, cd, cw):
    """Hurricane drag / wind terms (None winds: off); see include/fblts.h."""
    if uw_n is None or uw_t is None:
        _check(ctx, _lib_hurricane(ctx, None, None, 0.0, 0.0))
    else:
        a, b = _arr(uw_n, np.float64), _arr(uw_t, np.float64)
        _check_len(a, _sizes(ctx)[1], "uw_n")
        _check_len(b, _sizes(ctx)[1], "uw_t")
        _check(ctx, _lib_hurricane(ctx, _ptr(a, C.c_double), _ptr(b, C.c_double), float(cd), float(cw)))


def _host_ptr(x, n=None, what="buffer"):
    """numpy array or (pinned) CPU torch tensor -> (pointer, keepalive); n: required element count
    (checked here, so a short host buffer raises instead of being overrun by the C side)."""
    if isinstance(x, np.ndarray):
        a = _arr(x, np.float64)
        size = a.size
        p = (_ptr(a, C.c_double), a)
    else:
        if x.dtype != __import__("torch").float64 or x.device.type != "cpu" or not x.is_contiguous():
            raise ValueError("host buffers must be contiguous float64 CPU tensors or numpy arrays")
        size = x.numel()
        p = (C.cast(x.data_ptr(), _f64p), x)
    if n is not None and size != n:
        raise ValueError(f"{what}: {size} elements, expected {n}")
    return p


_MESH_SIZES = {}          # context handle -> (nCells, nEdges) of its uploaded (global) mesh


def _key(ctx):
    return ctx.value if isinstance(ctx, _vp) else ctx


def _sizes(ctx):
    """(nCells, nEdges) of the uploaded (global) mesh."""
    if _key(ctx) not in _MESH_SIZES:
        raise FbltsError(-8, "upload_mesh first (host buffer sizes unknown)")
    return _MESH_SIZES[_key(ctx)]


def _check_len(a, n, what):
    if a.size != n:
        raise ValueError(f"{what}: {a.size} elements, expected {n}")


def fblts_set_state(ctx, h, u, t=0.0):
    nC, nE = _sizes(ctx)
    ph, kh = _host_ptr(h, nC, "h")
    pu, ku = _host_ptr(u, nE, "u")
    _check(ctx, _lib_set_state(ctx, ph, pu, float(t)))


def fblts_set_vorticity(ctx, eta, nVertices):
    a = _arr(eta, np.float64)
    _check_len(a, nVertices, "eta")
    _check(ctx, _lib_set_vort(ctx, _ptr(a, C.c_double)))


def fblts_get_vorticity(ctx, nVertices):
    out = np.empty(nVertices)
    _check(ctx, _lib_get_vort(ctx, _ptr(out, C.c_double)))
    return out


def fblts_step(ctx, n_coarse):
    _check(ctx, _lib_step(ctx, int(n_coarse)))


def fblts_sync(ctx):
    _check(ctx, _lib_sync(ctx))


def fblts_get_state(ctx, h_out, u_out):
    """Fill host buffers (numpy arrays or CPU tensors) with the state; returns t."""
    nC, nE = _sizes(ctx)
    ph, kh = _host_ptr(h_out, nC, "h_out") if h_out is not None else (None, None)
    pu, ku = _host_ptr(u_out, nE, "u_out") if u_out is not None else (None, None)
    if isinstance(h_out, np.ndarray) and kh is not h_out or isinstance(u_out, np.ndarray) and ku is not u_out:
        raise ValueError("get_state needs contiguous float64 numpy outputs")
    t = C.c_double()
    _check(ctx, _lib_get_state(ctx, ph, pu, C.byref(t)))
    return t.value


def fblts_diagnostics(ctx):
    out = np.zeros(4)
    _check(ctx, _lib_diag(ctx, _ptr(out, C.c_double)))
    return out


def fblts_diagnostics_pv(ctx):
    out = np.zeros(1)
    _check(ctx, _lib_diag_pv(ctx, _ptr(out, C.c_double)))
    return float(out[0])


def fblts_diagnostics_mass(ctx):
    out = np.zeros(2)
    _check(ctx, _lib_diag_mass(ctx, _ptr(out, C.c_double)))
    return out


def fblts_diagnostics_async(ctx, out):
    """Enqueue the diagnostics of the current state; `out` (contiguous float64 numpy array of 4, kept
    alive by the caller) holds them after the next synchronising call."""
    if not (isinstance(out, np.ndarray) and out.dtype == np.float64 and out.size >= 4 and out.flags.c_contiguous):
        raise ValueError("diagnostics_async needs a contiguous float64 numpy array of 4")
    _check(ctx, _lib_diag_async(ctx, _ptr(out, C.c_double)))
    return out


def fblts_diagnostics_mass_async(ctx, out):
    """Enqueue (mass, min h) of the current state; `out` (contiguous float64 numpy array of 2, kept alive by
    the caller) holds them after the next synchronising call."""
    if not (isinstance(out, np.ndarray) and out.dtype == np.float64 and out.size >= 2 and out.flags.c_contiguous):
        raise ValueError("diagnostics_mass_async needs a contiguous float64 numpy array of 2")
    _check(ctx, _lib_diag_mass_async(ctx, _ptr(out, C.c_double)))
    return out


def fblts_profile(ctx, n_coarse):
    ms = np.zeros(NUM_KERNELS)
    cnt = np.zeros(NUM_KERNELS, np.int64)
    _check(ctx, _lib_profile(ctx, int(n_coarse), _ptr(ms, C.c_double), _ptr(cnt, C.c_int64)))
    return ms, cnt


def fblts_build_info():
    """Compile-time knobs of the loaded library as a dict, e.g. {"probe": "0", "check": "0", ...}."""
    return dict(kv.split("=", 1) for kv in _lib_build_info().decode().split())


def require_default_build():
    """Raise unless the loaded library is a measurement build (no FBLTS_PROBE work skipping, no
    FBLTS_CHECK bounds traps) -- bench.py calls this before timing anything."""
    info = fblts_build_info()
    if info.get("probe") != "0" or info.get("check") != "0":
        raise RuntimeError(f"libfblts.so is a development build ({info}); rebuild with "
                           "`python -m paper_2405_10505_b200.build --force` before measuring")
    return info


def fblts_kernel_name(kind):
    return _lib_kname(int(kind)).decode()


def fblts_last_error(ctx):
    return _lib_last_error(ctx).decode()


def fblts_destroy(ctx):
    _MESH_SIZES.pop(_key(ctx), None)
    _lib_destroy(ctx)
