"""B200-native (sm_100a) hot path of FoE-prior despeckling solved by iPiano (arXiv:1404.5344).

The product is libfoe.so (include/foe.h), hand-written CUDA for sm_100a; this package
is its thin ctypes binding (``foe``) plus the in-tree build (``_lib``).  PyTorch is used
only for device memory, streams and torch.distributed process groups.
"""
from . import _lib
from .foe import *  # noqa: F401,F403
from .foe import EXPORTED, Comm, FoeError, IPianoConfig, Model, Slabs, State, lib

__all__ = list(EXPORTED) + ["Comm", "FoeError", "IPianoConfig", "Model", "Slabs", "State", "lib", "build"]


def build(force: bool = False, verbose: bool = False) -> str:
    return _lib.build(force=force, verbose=verbose)
