"""B200-native FB-LTS hot path (arXiv 2405.10505): sm_100a CUDA kernels behind the C ABI
include/fblts.h, with a thin ctypes binding.  ``Solver`` needs a CUDA device; importing
the binding fails loudly if libfblts.so has not been built (no CPU fallback)."""

__all__ = ["Solver", "SolverGroup", "abi"]


def __getattr__(name):
    if name in ("Solver", "SolverGroup"):
        from . import solver
        return getattr(solver, name)
    if name == "abi":
        from . import _abi
        return _abi
    raise AttributeError(name)
