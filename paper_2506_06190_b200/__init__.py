"""NAT Helmholtz boundary-integral hot path on B200 (sm_100a).

The product is the C-ABI library ``libnat.so`` (``include/nat.h``) built from ``csrc/``;
``nat`` is its thin ctypes binding (same function names).  No CPU fallback exists.
"""
from . import nat  # noqa: F401
from .nat import NatError, Mesh, Geom, Sources  # noqa: F401
