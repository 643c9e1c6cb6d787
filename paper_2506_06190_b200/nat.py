"""Thin ctypes binding of libnat (include/nat.h).  Argument marshalling only: every step
of the hot path runs in the library's CUDA kernels.  torch supplies device memory and
streams.  There is no fallback: if libnat.so is missing or the device is not a CUDA
device, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import Optional, Sequence

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libnat.so")

NAT_OK, NAT_WARN_NOT_CONVERGED = 0, 1
NAT_FP32, NAT_FP64 = 0, 1
STATUS_NAMES = {0: "NAT_OK", 1: "NAT_WARN_NOT_CONVERGED", -1: "NAT_ERR_INVALID_ARG",
                -2: "NAT_ERR_CUDA", -3: "NAT_ERR_NCCL", -4: "NAT_ERR_SINGULAR",
                -5: "NAT_ERR_NUMERIC", -6: "NAT_ERR_WORKSPACE"}


class NatError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {message}")
        self.status = status


class _Mesh(C.Structure):
    _fields_ = [("n_vert", C.c_int64), ("n_tri", C.c_int64), ("vxyz", C.c_void_p),
                ("tri", C.c_void_p)]


class _Geom(C.Structure):
    _fields_ = [("n_tri", C.c_int64), ("centroid", C.c_void_p), ("normal", C.c_void_p),
                ("area", C.c_void_p), ("diam", C.c_void_p), ("area_cdf", C.c_void_p),
                ("total_area", C.c_double), ("center", C.c_double * 3),
                ("bound_radius", C.c_double), ("volume", C.c_double)]


class _QuadOpts(C.Structure):
    _fields_ = [("far_pts", C.c_int), ("near_levels_S", C.c_int), ("near_levels_N", C.c_int),
                ("near_eta", C.c_double), ("self_theta_pts", C.c_int), ("burton_miller", C.c_int),
                ("galerkin", C.c_int), ("ss_order", C.c_int)]


class _SolveInfo(C.Structure):
    _fields_ = [("iters", C.c_int), ("converged", C.c_int), ("rel_residual", C.c_double),
                ("t_total_s", C.c_double), ("t_matvec_s", C.c_double), ("t_comm_s", C.c_double)]


class _BemMf(C.Structure):
    _fields_ = [("mesh", C.POINTER(_Mesh)), ("geom", C.POINTER(_Geom)), ("opts", C.POINTER(_QuadOpts)),
                ("k", C.c_double), ("prec", C.c_int), ("row_begin", C.c_int64), ("row_end", C.c_int64),
                ("near_row_ptr", C.c_void_p), ("near_col", C.c_void_p), ("near_cls", C.c_void_p),
                ("nnz", C.c_int64), ("near_delta", C.c_void_p), ("diag_delta", C.c_void_p)]


class _McOpts(C.Structure):
    _fields_ = [("M", C.c_int64), ("seed", C.c_uint64), ("stream_id", C.c_uint64),
                ("eps", C.c_double), ("samples_in", C.c_void_p), ("sample_tri_in", C.c_void_p)]


class _NfConfig(C.Structure):
    _fields_ = [("n_v", C.c_int), ("n_out", C.c_int)]


class _Sources(C.Structure):
    _fields_ = [("n_src", C.c_int64), ("xyz", C.c_void_p), ("nrm", C.c_void_p),
                ("w", C.c_void_p), ("n_modes", C.c_int), ("p", C.c_void_p), ("g", C.c_void_p),
                ("center", C.c_double * 3)]


_P = C.c_void_p
_I64 = C.c_int64
_D = C.c_double
_SZ = C.c_size_t
# name -> (restype, argtypes)
_SIGS = {
    "nat_abi_version": (C.c_int, []),
    "nat_last_error": (C.c_char_p, []),
    "nat_mesh_prepare_workspace": (_SZ, [_I64, _I64]),
    "nat_mesh_prepare": (C.c_int, [C.POINTER(_Mesh), C.POINTER(_Geom), _P, _SZ, _P]),
    "nat_bem_near_workspace": (_SZ, [_I64]),
    "nat_bem_near_count": (C.c_int, [C.POINTER(_Mesh), C.POINTER(_Geom), C.POINTER(_QuadOpts),
                                     _I64, _I64, _P, C.POINTER(_I64), _P, _SZ, _P]),
    "nat_bem_near_build": (C.c_int, [C.POINTER(_Mesh), C.POINTER(_Geom), C.POINTER(_QuadOpts),
                                     _I64, _I64, _P, _P, _P, _P, _SZ, _P]),
    "nat_bem_assemble_workspace": (_SZ, [_I64, _I64, _I64, C.c_int]),
    "nat_bem_assemble": (C.c_int, [C.POINTER(_Mesh), C.POINTER(_Geom), C.POINTER(_QuadOpts),
                                   _P, _P, _P, _I64, _D, C.c_int, _I64, _I64, C.c_int, _P, _P, _I64,
                                   _P, _P, _SZ, _P]),
    "nat_bem_assemble_multi_workspace": (_SZ, [_I64, _I64, _I64, C.c_int, C.c_int]),
    "nat_bem_assemble_multi": (C.c_int, [C.POINTER(_Mesh), C.POINTER(_Geom), C.POINTER(_QuadOpts),
                                         _P, _P, _P, _I64, C.c_int, C.POINTER(_D), C.c_int, _I64, _I64, C.c_int,
                                         _P, C.POINTER(_P), _I64, _P, _P, _SZ, _P]),
    "nat_bem_matvec": (C.c_int, [C.c_int, _I64, _I64, _P, _I64, _P, _P, _P]),
    "nat_bem_mf_workspace": (_SZ, [C.POINTER(_BemMf), _I64, C.c_int]),
    "nat_bem_mf_prepare": (C.c_int, [C.POINTER(_BemMf), C.c_int, _P, _P, _P, _SZ, _P]),
    "nat_bem_mf_matvec": (C.c_int, [C.POINTER(_BemMf), _P, _P, _P, _SZ, _P]),
    "nat_bem_mf_solve_workspace": (_SZ, [C.POINTER(_BemMf), C.c_int, C.c_int]),
    "nat_bem_mf_solve": (C.c_int, [_P, C.POINTER(_BemMf), _P, _P, _D, C.c_int, _P, _SZ, C.POINTER(_SolveInfo),
                                   _P]),
    "nat_kernel_timer_enable": (None, [C.c_int]),
    "nat_kernel_timer_read": (C.c_int, [C.c_int, C.POINTER(_D), C.POINTER(_D), C.POINTER(_I64)]),
    "nat_kernel_timer_read_modes": (C.c_int, [C.c_int, C.c_int, C.POINTER(_D), C.POINTER(_D), C.POINTER(_I64)]),
    "nat_comm_unique_id": (C.c_int, [_P]),
    "nat_comm_create_from_id": (C.c_int, [C.POINTER(_P), _P, C.c_int, C.c_int]),
    "nat_comm_create": (C.c_int, [C.POINTER(_P), _P, C.c_int, C.c_int]),
    "nat_comm_destroy": (C.c_int, [_P]),
    "nat_comm_create_host": (C.c_int, [C.POINTER(_P), C.c_int, C.c_int, _P, _P]),
    "nat_bem_solve_workspace": (_SZ, [C.c_int, _I64, _I64, C.c_int]),
    "nat_bem_solve": (C.c_int, [_P, C.c_int, _I64, _I64, _I64, _P, _I64, _P, _P, _D, C.c_int,
                                _P, _SZ, C.POINTER(_SolveInfo), _P]),
    "nat_mc_set_groups": (C.c_int, [C.c_int]),
    "nat_krylov_config": (C.c_int, [C.c_int, C.c_int, C.c_int]),
    "nat_mc_sample": (C.c_int, [C.POINTER(_Mesh), C.POINTER(_Geom), _I64, C.c_uint64,
                                C.c_uint64, _P, _P, _P]),
    "nat_mc_op_workspace": (_SZ, [C.c_int, _I64, C.c_int]),
    "nat_mc_rhs": (C.c_int, [C.c_int, _I64, _P, C.c_int, C.POINTER(_D), _P, _D, _D, _P, _P,
                             _SZ, _P]),
    "nat_mc_apply": (C.c_int, [C.c_int, _I64, _P, C.c_int, C.POINTER(_D), _P, _D, _D, _P, _P, _SZ,
                               _P]),
    "nat_mc_check_coincident": (C.c_int, [_I64, _P, C.POINTER(_I64), _P, _SZ, _P]),
    "nat_mc_gather_neumann": (C.c_int, [C.c_int, _I64, _I64, _P, _P, _P, _P]),
    "nat_mc_workspace": (_SZ, [C.c_int, _I64, C.c_int, C.c_int]),
    "nat_mc_surface_pressure": (C.c_int, [C.POINTER(_Mesh), C.POINTER(_Geom), C.c_int,
                                          C.POINTER(_D), _P, C.POINTER(_McOpts), C.c_int, _D,
                                          C.c_int, _P, _P, _P, _P, _SZ, C.POINTER(_SolveInfo),
                                          _P]),
    "nat_mc_rows_workspace": (_SZ, [C.c_int, _I64, C.c_int, _I64]),
    "nat_mc_apply_rows": (C.c_int, [C.c_int, _I64, _P, C.c_int, C.POINTER(_D), _P, _D, _D, _I64, _I64, _P, _P, _SZ,
                                    _P]),
    "nat_mc_sharded_workspace": (_SZ, [C.c_int, _I64, C.c_int, C.c_int, C.c_int]),
    "nat_mc_surface_pressure_sharded": (C.c_int, [_P, C.POINTER(_Mesh), C.POINTER(_Geom), C.c_int, C.POINTER(_D), _P,
                                                  C.POINTER(_McOpts), C.c_int, _D, C.c_int, _P, _P, _P, _P, _SZ,
                                                  C.POINTER(_SolveInfo), _P]),
    "nat_bem_sources": (C.c_int, [C.POINTER(_Mesh), C.POINTER(_Geom), C.c_int, C.c_int, _P, _P,
                                  _P, _P, _P, _P, _P, _P]),
    "nat_mc_sources": (C.c_int, [_I64, _P, _D, _P, _P, _P, _P]),
    "nat_radiate_workspace": (_SZ, [C.c_int, _I64, C.c_int, _I64]),
    "nat_radiate_field": (C.c_int, [C.POINTER(_Sources), C.c_int, C.POINTER(_D), _I64, _P, _P,
                                    _P, _SZ, _P]),
    "nat_listener_grid": (C.c_int, [C.POINTER(_D), _D, C.c_int, C.c_int, C.c_int, _D, _D, _P,
                                    _P]),
    "nat_mc_poisson_workspace": (_SZ, [C.POINTER(_Geom), _I64, _D]),
    "nat_mc_poisson_sample": (C.c_int, [C.POINTER(_Mesh), C.POINTER(_Geom), _I64, _D, C.c_uint64, C.c_uint64,
                                        _P, _P, _I64, C.POINTER(_I64), C.POINTER(_D), _P, _SZ, _P]),
    "nat_listener_random_shell": (C.c_int, [C.POINTER(_D), _D, _I64, _D, _D, C.c_uint64, C.c_uint64, _P,
                                            _P]),
    "nat_nf_param_count": (_I64, [C.POINTER(_NfConfig)]),
    "nat_nf_workspace": (_SZ, [C.POINTER(_NfConfig), _I64]),
    "nat_nf_forward": (C.c_int, [C.POINTER(_NfConfig), _P, _I64, _P, _P, _P, _SZ, _P]),
    "nat_nf_train_step": (C.c_int, [C.POINTER(_NfConfig), _P, _P, _P, C.c_int, C.c_float, _I64, _P, _P, _P, _P, _P,
                                    _SZ, _P]),
    "nat_nf_gemm_bf16": (C.c_int, [_I64, _I64, _I64, _P, _I64, C.c_int, _P, _I64, C.c_int, _P, _I64, _P]),
}

_lib = None


def lib():
    """Load libnat.so (raises if absent: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2506_06190_b200.build`")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


# Concurrent-sweep configuration (the C4 sweep runs SWEEP_WORKERS geometries at once on one
# GPU, each on its own stream): the fused Arnoldi step uses clusters of two 256-thread CTAs
# per system without the shared-memory residency cap, so its latency-bound clusters
# co-reside with the pair kernels of the other streams instead of holding whole SMs (bench
# A/B on B200: 2.77 -> 2.70 -> 2.625 s per 64-geometry step).  Library defaults (one solve at a time) are unchanged; the settings are
# read once, at the first solve of the process.
SWEEP_WORKERS = 6


def sweep_tuning():
    """The C4 sweep's configuration (many geometries in flight on one GPU)."""
    nat_krylov_config(2, 256, 0)   # 2 x 256-thread CTAs per system, no cap (2.657 -> 2.625 s per step)
    nat_mc_set_groups(1)           # the workers already overlap whole geometries


def single_call_tuning():
    """The library defaults, for one large solve at a time (C3): wide fused step, two groups."""
    nat_krylov_config(4, 512, 120)
    nat_mc_set_groups(2)


def exported_symbols():
    return list(_SIGS)


def _check(status, allow_warn=False):
    if status == NAT_OK or (allow_warn and status == NAT_WARN_NOT_CONVERGED):
        return status
    raise NatError(status, lib().nat_last_error().decode())


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_cuda:
        raise NatError(-1, "tensor must live on a CUDA device")
    if not t.is_contiguous():
        raise NatError(-1, "tensor must be contiguous")
    return C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ws(nbytes: int, device):
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def _prec(prec):
    if prec in ("fp32", NAT_FP32, torch.float32):
        return NAT_FP32
    if prec in ("fp64", NAT_FP64, torch.float64):
        return NAT_FP64
    raise ValueError(f"bad precision {prec!r}")


# ------------------------------------------------------------------------------------
# data holders
# ------------------------------------------------------------------------------------
@dataclasses.dataclass
class Mesh:
    vxyz: torch.Tensor  # (3, V) float64 cuda
    tri: torch.Tensor   # (3, N) int32 cuda

    @classmethod
    def from_numpy(cls, v, t, device="cuda"):
        v = np.ascontiguousarray(np.asarray(v, dtype=np.float64).T)
        t = np.ascontiguousarray(np.asarray(t, dtype=np.int32).T)
        return cls(torch.from_numpy(v).to(device), torch.from_numpy(t).to(device))

    @property
    def n_vert(self):
        return self.vxyz.shape[1]

    @property
    def n_tri(self):
        return self.tri.shape[1]

    def c(self):
        return _Mesh(self.n_vert, self.n_tri, _ptr(self.vxyz), _ptr(self.tri))


@dataclasses.dataclass
class Geom:
    centroid: torch.Tensor
    normal: torch.Tensor
    area: torch.Tensor
    diam: torch.Tensor
    area_cdf: torch.Tensor
    total_area: float = 0.0
    center: tuple = (0.0, 0.0, 0.0)
    bound_radius: float = 0.0
    volume: float = 0.0

    def c(self):
        g = _Geom(self.area.shape[0], _ptr(self.centroid), _ptr(self.normal), _ptr(self.area),
                  _ptr(self.diam), _ptr(self.area_cdf), self.total_area, (C.c_double * 3)(*self.center),
                  self.bound_radius, self.volume)
        return g


@dataclasses.dataclass
class Sources:
    xyz: torch.Tensor     # (3, S) float64
    nrm: torch.Tensor     # (3, S) float64
    w: torch.Tensor       # (S,) float64
    p: torch.Tensor       # (n_modes, S) complex128
    g: torch.Tensor       # (n_modes, S) complex128
    center: tuple = (0.0, 0.0, 0.0)

    def c(self):
        return _Sources(self.xyz.shape[1], _ptr(self.xyz), _ptr(self.nrm), _ptr(self.w),
                        self.p.shape[0], _ptr(self.p), _ptr(self.g), (C.c_double * 3)(*self.center))


def quad_opts(far_pts=0, near_levels_S=0, near_levels_N=0, near_eta=0.0, self_theta_pts=0, burton_miller=False,
              galerkin=False, ss_order=0):
    """nat_quad_opts (zeros = defaults); burton_miller selects Eq. BM with beta = i/k (NEXT-1);
    galerkin the P0 Galerkin discretisation with Sauter-Schwab singular quadrature (NEXT-2)."""
    return _QuadOpts(far_pts, near_levels_S, near_levels_N, near_eta, self_theta_pts, int(bool(burton_miller)),
                     int(bool(galerkin)), int(ss_order))


# ------------------------------------------------------------------------------------
# calls (same names as the C ABI)
# ------------------------------------------------------------------------------------
def nat_abi_version():
    return lib().nat_abi_version()


def nat_mesh_prepare(mesh: Mesh) -> Geom:
    dev = mesh.vxyz.device
    n = mesh.n_tri
    f = dict(dtype=torch.float64, device=dev)
    geo = Geom(torch.empty(3, n, **f), torch.empty(3, n, **f), torch.empty(n, **f),
               torch.empty(n, **f), torch.empty(n, **f))
    cg = geo.c()
    ws = _ws(lib().nat_mesh_prepare_workspace(mesh.n_vert, n), dev)
    _check(lib().nat_mesh_prepare(C.byref(mesh.c()), C.byref(cg), _ptr(ws), ws.numel(), _stream()))
    geo.total_area, geo.center = cg.total_area, tuple(cg.center)
    geo.bound_radius, geo.volume = cg.bound_radius, cg.volume
    return geo


def nat_listener_grid(center, R, n_theta, n_phi, n_r, r_lo=1.5, r_hi=3.0, device="cuda", out=None):
    n = n_theta * n_phi * n_r
    out = torch.empty(3, n, dtype=torch.float64, device=device) if out is None else out
    c = (C.c_double * 3)(*[float(x) for x in center])
    _check(lib().nat_listener_grid(c, float(R), n_theta, n_phi, n_r, float(r_lo), float(r_hi),
                                   _ptr(out), _stream()))
    return out


def nat_listener_random_shell(center, R, n, r_lo=1.5, r_hi=3.0, seed=0, stream_id=0, device="cuda"):
    """n listener points uniform in the volume of the shell R r_lo <= |x - c| <= R r_hi
    (Philox tag 1; reading R-listen-rand).  Returns (3, n) float64."""
    out = torch.empty(3, n, dtype=torch.float64, device=device)
    c = (C.c_double * 3)(*[float(x) for x in center])
    _check(lib().nat_listener_random_shell(c, float(R), int(n), float(r_lo), float(r_hi), int(seed),
                                           int(stream_id), _ptr(out), _stream()))
    return out


def nat_bem_sources(mesh: Mesh, geom: Geom, p_tri, g_tri, q_rad=3) -> Sources:
    dev = mesh.vxyz.device
    p_tri = torch.atleast_2d(p_tri).to(torch.complex128).contiguous()
    g_tri = torch.atleast_2d(g_tri).to(torch.complex128).contiguous()
    nm = p_tri.shape[0]
    S = mesh.n_tri * q_rad
    f = dict(dtype=torch.float64, device=dev)
    src = Sources(torch.empty(3, S, **f), torch.empty(3, S, **f), torch.empty(S, **f),
                  torch.empty(nm, S, dtype=torch.complex128, device=dev),
                  torch.empty(nm, S, dtype=torch.complex128, device=dev), tuple(geom.center))
    _check(lib().nat_bem_sources(C.byref(mesh.c()), C.byref(geom.c()), q_rad, nm, _ptr(p_tri),
                                 _ptr(g_tri), _ptr(src.xyz), _ptr(src.nrm), _ptr(src.w),
                                 _ptr(src.p), _ptr(src.g), _stream()))
    return src


def nat_mc_sources(samples, total_area, p, g, center=(0.0, 0.0, 0.0)) -> Sources:
    dev = samples.device
    M = samples.shape[1]
    f = dict(dtype=torch.float64, device=dev)
    src = Sources(torch.empty(3, M, **f), torch.empty(3, M, **f), torch.empty(M, **f),
                  torch.atleast_2d(p).to(torch.complex128).contiguous(),
                  torch.atleast_2d(g).to(torch.complex128).contiguous(), tuple(center))
    _check(lib().nat_mc_sources(M, _ptr(samples), float(total_area), _ptr(src.xyz), _ptr(src.nrm),
                                _ptr(src.w), _stream()))
    return src


class RadiatePlan:
    """Pre-sized workspace for repeated nat_radiate_field calls (bench / serving loop)."""

    def __init__(self, n_src, n_modes, n_lis, prec="fp32", device="cuda"):
        self.prec = _prec(prec)
        self.ws = _ws(lib().nat_radiate_workspace(self.prec, n_src, n_modes, n_lis), device)


def nat_radiate_field(src: Sources, k: Sequence[float], lis_xyz: torch.Tensor, prec="fp32",
                      out: Optional[torch.Tensor] = None, plan: Optional[RadiatePlan] = None):
    pr = _prec(prec)
    nm = src.p.shape[0]
    k = np.ascontiguousarray(np.atleast_1d(np.asarray(k, dtype=np.float64)))
    if k.size != nm:
        raise NatError(-1, f"{k.size} wavenumbers for {nm} modes")
    n_lis = lis_xyz.shape[1]
    dev = lis_xyz.device
    if out is None:
        out = torch.empty(nm, n_lis, dtype=torch.complex128, device=dev)
    ws = plan.ws if plan is not None else _ws(
        lib().nat_radiate_workspace(pr, src.xyz.shape[1], nm, n_lis), dev)
    _check(lib().nat_radiate_field(C.byref(src.c()), pr, k.ctypes.data_as(C.POINTER(C.c_double)),
                                   n_lis, _ptr(lis_xyz), _ptr(out), _ptr(ws), ws.numel(),
                                   _stream()))
    return out


# ------------------------------------------------------------------------------------
# dense BEM (rows a2, a4-a7)
# ------------------------------------------------------------------------------------
@dataclasses.dataclass
class NearList:
    row_begin: int
    row_end: int
    row_ptr: torch.Tensor  # (rows+1,) int64
    col: torch.Tensor      # (nnz,) int32
    cls: torch.Tensor      # (nnz,) uint8

    @property
    def nnz(self):
        return self.col.numel()


def nat_bem_near_list(mesh: Mesh, geom: Geom, row_begin=0, row_end=None, opts=None) -> NearList:
    """nat_bem_near_count + nat_bem_near_build."""
    row_end = mesh.n_tri if row_end is None else row_end
    dev = mesh.vxyz.device
    o = opts or quad_opts()
    rp = torch.empty(row_end - row_begin + 1, dtype=torch.int64, device=dev)
    ws = _ws(lib().nat_bem_near_workspace(mesh.n_tri), dev)
    nnz = C.c_int64(0)
    _check(lib().nat_bem_near_count(C.byref(mesh.c()), C.byref(geom.c()), C.byref(o), row_begin,
                                    row_end, _ptr(rp), C.byref(nnz), _ptr(ws), ws.numel(), _stream()))
    col = torch.empty(max(nnz.value, 1), dtype=torch.int32, device=dev)[: nnz.value]
    cls = torch.empty(max(nnz.value, 1), dtype=torch.uint8, device=dev)[: nnz.value]
    _check(lib().nat_bem_near_build(C.byref(mesh.c()), C.byref(geom.c()), C.byref(o), row_begin,
                                    row_end, _ptr(rp), C.c_void_p(col.data_ptr()),
                                    C.c_void_p(cls.data_ptr()), _ptr(ws), ws.numel(), _stream()))
    return NearList(row_begin, row_end, rp, col, cls)


def nat_bem_assemble(mesh: Mesh, geom: Geom, near: NearList, k: float, g=None, prec="fp32",
                     opts=None, A: Optional[torch.Tensor] = None, lda: Optional[int] = None,
                     rhs: Optional[torch.Tensor] = None):
    """Rows [near.row_begin, near.row_end) of A (c64 for fp32, c128 for fp64) and
    rhs = -V g (c128 [n_rhs][rows]).  Returns (A, rhs)."""
    pr = _prec(prec)
    dev = mesh.vxyz.device
    n = mesh.n_tri
    rows = near.row_end - near.row_begin
    lda = lda or (n + (n & 1))
    cdt = torch.complex64 if pr == NAT_FP32 else torch.complex128
    if A is None:
        A = torch.empty(rows, lda, dtype=cdt, device=dev)
    n_rhs = 0
    if g is None:
        rhs = None
    else:
        g = torch.atleast_2d(g).to(torch.complex128).contiguous()
        n_rhs = g.shape[0]
        if rhs is None:
            rhs = torch.empty(n_rhs, rows, dtype=torch.complex128, device=dev)
    o = opts or quad_opts()
    ws = _ws(lib().nat_bem_assemble_workspace(n, rows, near.nnz, n_rhs), dev)
    _check(lib().nat_bem_assemble(C.byref(mesh.c()), C.byref(geom.c()), C.byref(o), _ptr(near.row_ptr),
                                  C.c_void_p(near.col.data_ptr()), C.c_void_p(near.cls.data_ptr()),
                                  int(near.nnz), float(k), pr, near.row_begin, near.row_end, n_rhs, _ptr(g), _ptr(A),
                                  lda, _ptr(rhs), _ptr(ws), ws.numel(), _stream()))
    return A, rhs


def nat_bem_assemble_multi(mesh: Mesh, geom: Geom, near: NearList, ks, g=None, prec="fp32", opts=None,
                           A=None, lda: Optional[int] = None, rhs: Optional[torch.Tensor] = None, ws=None):
    """a4 + a5 for several wavenumbers in one call (one far pass for all of them on the fp32
    collocation path).  Returns (list of A, rhs c128 [n_k][n_rhs][rows] or None)."""
    pr = _prec(prec)
    dev = mesh.vxyz.device
    n = mesh.n_tri
    rows = near.row_end - near.row_begin
    lda = lda or (n + (n & 1))
    ks, kp = _karr(ks)
    nk = ks.size
    cdt = torch.complex64 if pr == NAT_FP32 else torch.complex128
    if A is None:
        A = [torch.empty(rows, lda, dtype=cdt, device=dev) for _ in range(nk)]
    n_rhs = 0
    if g is not None:
        g = torch.atleast_2d(g).to(torch.complex128).contiguous()
        n_rhs = g.shape[0]
        if rhs is None:
            rhs = torch.empty(nk, n_rhs, rows, dtype=torch.complex128, device=dev)
    else:
        rhs = None
    o = opts or quad_opts()
    if ws is None:
        ws = _ws(lib().nat_bem_assemble_multi_workspace(n, rows, near.nnz, n_rhs, nk), dev)
    ptrs = (C.c_void_p * nk)(*[a.data_ptr() for a in A])
    for a in A:
        _ptr(a)
    _check(lib().nat_bem_assemble_multi(C.byref(mesh.c()), C.byref(geom.c()), C.byref(o), _ptr(near.row_ptr),
                                        C.c_void_p(near.col.data_ptr()), C.c_void_p(near.cls.data_ptr()),
                                        int(near.nnz), nk, kp, pr, near.row_begin, near.row_end, n_rhs, _ptr(g),
                                        ptrs, lda, _ptr(rhs), _ptr(ws), ws.numel(), _stream()))
    return A, rhs


def nat_bem_matvec(A: torch.Tensor, x: torch.Tensor, n: Optional[int] = None, out=None):
    pr = NAT_FP32 if A.dtype == torch.complex64 else NAT_FP64
    rows, lda = A.shape
    n = n or x.numel()
    out = torch.empty(rows, dtype=torch.complex128, device=A.device) if out is None else out
    _check(lib().nat_bem_matvec(pr, rows, n, _ptr(A), lda, _ptr(x.to(torch.complex128).contiguous()),
                                _ptr(out), _stream()))
    return out


_AllGatherFn = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_size_t, C.c_int, C.c_int)


class Comm:
    """NCCL communicator built from a torch.distributed-broadcast unique id (or, for tests
    of the world > 1 path on one GPU, the host-staged backend over a gloo group)."""

    def __init__(self, rank: int, world: int, uid: Optional[bytes] = None, nccl_comm: Optional[int] = None,
                 _host_fn=None):
        self.rank, self.world = rank, world
        self.handle = C.c_void_p()
        if _host_fn is not None:   # nat_comm_create_host (keeps the callback alive)
            self._cb = _AllGatherFn(_host_fn)
            _check(lib().nat_comm_create_host(C.byref(self.handle), rank, world, C.cast(self._cb, C.c_void_p), None))
            return
        if uid is None:   # borrow a caller-owned ncclComm_t (or none: world 1)
            _check(lib().nat_comm_create(C.byref(self.handle), C.c_void_p(nccl_comm), rank, world))
            return
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        _check(lib().nat_comm_create_from_id(C.byref(self.handle), buf, rank, world))

    @classmethod
    def borrow(cls, nccl_comm: Optional[int], rank: int = 0, world: int = 1):
        """Wraps an existing ncclComm_t (address as int; None => single rank); never destroyed here."""
        return cls(rank, world, None, nccl_comm)

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _check(lib().nat_comm_unique_id(buf))
        return bytes(buf)

    @staticmethod
    def broadcast_unique_id(make_id=None) -> bytes:
        """Rank 0's 128-byte NCCL unique id, broadcast with torch.distributed (works on
        nccl and gloo process groups)."""
        import torch.distributed as dist
        dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
        t = torch.zeros(128, dtype=torch.uint8, device=dev)
        if dist.get_rank() == 0:
            uid = (make_id or Comm.unique_id)()
            t.copy_(torch.frombuffer(bytearray(uid), dtype=torch.uint8))
        dist.broadcast(t, 0)
        return bytes(t.cpu().numpy().tobytes())

    @classmethod
    def host(cls, group=None):
        """Host-staged communicator: every all-gather of the library runs as
        torch.distributed.all_gather on `group` (e.g. gloo) over a pinned host buffer.  No
        kernel waits on another rank, so several ranks may share one GPU (tests)."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)

        def fn(user, buf, count, rk, ws):
            try:
                arr = np.ctypeslib.as_array(buf, shape=(int(count) * ws,))
                t = torch.from_numpy(arr)
                parts = [t[r * count:(r + 1) * count] for r in range(ws)]
                mine = parts[rk].clone()
                dist.all_gather(parts, mine, group=group)
                return 0
            except Exception:  # reported by the library as NAT_ERR_NCCL
                return 1

        return cls(rank, world, _host_fn=fn)

    @classmethod
    def from_torch_distributed(cls):
        import torch.distributed as dist
        return cls(dist.get_rank(), dist.get_world_size(), cls.broadcast_unique_id())

    def close(self):
        if self.handle:
            _check(lib().nat_comm_destroy(self.handle))
            self.handle = C.c_void_p()


# ------------------------------------------------------------------------------------
# Monte-Carlo BEM (rows a8-a10)
# ------------------------------------------------------------------------------------
def _karr(k):
    k = np.ascontiguousarray(np.atleast_1d(np.asarray(k, dtype=np.float64)))
    return k, k.ctypes.data_as(C.POINTER(C.c_double))


def nat_mc_sample(mesh: Mesh, geom: Geom, M: int, seed: int, stream_id: int = 0):
    """Returns (samples (6, M) float64 [xyz; normal], sample_tri (M,) int32)."""
    dev = mesh.vxyz.device
    smp = torch.empty(6, M, dtype=torch.float64, device=dev)
    tri = torch.empty(M, dtype=torch.int32, device=dev)
    _check(lib().nat_mc_sample(C.byref(mesh.c()), C.byref(geom.c()), M, seed, stream_id, _ptr(smp),
                               _ptr(tri), _stream()))
    return smp, tri


def nat_mc_check_coincident(samples: torch.Tensor):
    M = samples.shape[1]
    pair = (C.c_int64 * 2)()
    ws = _ws(256, samples.device)
    _check(lib().nat_mc_check_coincident(M, _ptr(samples), pair, _ptr(ws), ws.numel(), _stream()))
    return None


def nat_mc_gather_neumann(g_tri: torch.Tensor, sample_tri: torch.Tensor, out=None):
    g_tri = torch.atleast_2d(g_tri).to(torch.complex128).contiguous()
    n_sys, n_tri = g_tri.shape
    M = sample_tri.numel()
    out = torch.empty(n_sys, M, dtype=torch.complex128, device=g_tri.device) if out is None else out
    _check(lib().nat_mc_gather_neumann(n_sys, M, n_tri, _ptr(g_tri), _ptr(sample_tri), _ptr(out), _stream()))
    return out


def nat_mc_poisson_sample(mesh: Mesh, geom: Geom, M_target: int, seed: int = 0, stream_id: int = 0, r: float = 0.0):
    """Poisson-disk boundary samples (NEXT-3, reading R-poisson).  Returns (samples (6, M)
    float64, sample_tri (M,) int32, r)."""
    dev = mesh.vxyz.device
    gc = geom.c()
    ws = _ws(lib().nat_mc_poisson_workspace(C.byref(gc), int(M_target), float(r)), dev)
    cap = 2 * int(M_target) + 16
    smp = torch.empty(6 * cap, dtype=torch.float64, device=dev)
    tri = torch.empty(cap, dtype=torch.int32, device=dev)
    M = C.c_int64(0)
    rr = C.c_double(0.0)
    _check(lib().nat_mc_poisson_sample(C.byref(mesh.c()), C.byref(gc), int(M_target), float(r), int(seed),
                                       int(stream_id), _ptr(smp), _ptr(tri), cap, C.byref(M), C.byref(rr),
                                       _ptr(ws), ws.numel(), _stream()))
    M = M.value
    return smp[: 6 * M].view(6, M), tri[:M], rr.value


def nat_mc_rhs(samples, k, g, total_area, eps=0.0, prec="fp32"):
    """a9 right-hand sides; the library derives eps (unless eps > 0) and w from total_area."""
    pr = _prec(prec)
    M = samples.shape[1]
    g = torch.atleast_2d(g).to(torch.complex128).contiguous()
    ks, kp = _karr(k)
    b = torch.empty_like(g)
    ws = _ws(lib().nat_mc_op_workspace(pr, M, g.shape[0]), samples.device)
    _check(lib().nat_mc_rhs(pr, M, _ptr(samples), g.shape[0], kp, _ptr(g), float(total_area), float(eps), _ptr(b),
                            _ptr(ws), ws.numel(), _stream()))
    return b


def nat_mc_apply(samples, k, p, total_area, eps=0.0, prec="fp32"):
    """a10 operator applied to p; eps (unless > 0) and w derived from total_area by the library."""
    pr = _prec(prec)
    M = samples.shape[1]
    p = torch.atleast_2d(p).to(torch.complex128).contiguous()
    ks, kp = _karr(k)
    out = torch.empty_like(p)
    ws = _ws(lib().nat_mc_op_workspace(pr, M, p.shape[0]), samples.device)
    _check(lib().nat_mc_apply(pr, M, _ptr(samples), p.shape[0], kp, _ptr(p), float(total_area), float(eps), _ptr(out), _ptr(ws),
                              ws.numel(), _stream()))
    return out


class McPlan:
    """Pre-sized workspace for repeated nat_mc_surface_pressure calls."""

    def __init__(self, M, n_sys, prec="fp32", max_iter=200, device="cuda"):
        self.prec = _prec(prec)
        self.ws = _ws(lib().nat_mc_workspace(self.prec, M, n_sys, max_iter), device)


def nat_mc_surface_pressure(mesh: Mesh, geom: Geom, k, g_tri, M: int, seed: int = 0, stream_id: int = 0,
                            eps: float = 0.0, prec="fp32", tol=1e-6, max_iter=200, samples_in=None,
                            sample_tri_in=None, plan: Optional[McPlan] = None, out=None):
    """Returns (samples (6, M), sample_tri (M,), p (n_sys, M) c128, infos list)."""
    pr = _prec(prec)
    dev = mesh.vxyz.device
    g_tri = torch.atleast_2d(g_tri).to(torch.complex128).contiguous()
    ks, kp = _karr(k)
    n_sys = ks.size
    if g_tri.shape[0] != n_sys:
        raise NatError(-1, f"{g_tri.shape[0]} Neumann fields for {n_sys} wavenumbers")
    if out is None:
        smp = torch.empty(6, M, dtype=torch.float64, device=dev)
        tri = torch.empty(M, dtype=torch.int32, device=dev)
        p = torch.empty(n_sys, M, dtype=torch.complex128, device=dev)
    else:
        smp, tri, p = out
    opts = _McOpts(M, seed, stream_id, float(eps), _ptr(samples_in), _ptr(sample_tri_in))
    ws = plan.ws if plan is not None else _ws(lib().nat_mc_workspace(pr, M, n_sys, max_iter), dev)
    infos = (_SolveInfo * n_sys)()
    st = lib().nat_mc_surface_pressure(C.byref(mesh.c()), C.byref(geom.c()), n_sys, kp, _ptr(g_tri),
                                       C.byref(opts), pr, float(tol), int(max_iter), _ptr(smp), _ptr(tri),
                                       _ptr(p), _ptr(ws), ws.numel(), infos, _stream())
    _check(st, allow_warn=True)
    return smp, tri, p, [dict(iters=i.iters, converged=i.converged, rel_residual=i.rel_residual,
                              t_total_s=i.t_total_s, t_matvec_s=i.t_matvec_s) for i in infos]


def nat_mc_apply_rows(samples, k, p, total_area, eps, row_begin: int, row_end: int, prec="fp32"):
    """Rows [row_begin, row_end) of the MC operator applied to p (n_sys, M) -> (n_sys, rows)."""
    pr = _prec(prec)
    M = samples.shape[1]
    ks, kp = _karr(k)
    p = torch.atleast_2d(p).to(torch.complex128).contiguous()
    rows = max(int(row_end) - int(row_begin), 1)   # the library validates the range
    out = torch.empty(ks.size, rows, dtype=torch.complex128, device=samples.device)
    ws = _ws(lib().nat_mc_rows_workspace(pr, M, ks.size, rows), samples.device)
    _check(lib().nat_mc_apply_rows(pr, M, _ptr(samples), ks.size, kp, _ptr(p), float(total_area), float(eps), int(row_begin),
                                   int(row_end), _ptr(out), _ptr(ws), ws.numel(), _stream()))
    return out


def nat_mc_surface_pressure_sharded(mesh: Mesh, geom: Geom, k, g_tri, M: int, comm: Optional["Comm"] = None,
                                    seed: int = 0, stream_id: int = 0, eps: float = 0.0, prec="fp32", tol=1e-6,
                                    max_iter=200, samples_in=None, sample_tri_in=None, out=None, ws=None):
    """nat_mc_surface_pressure row-sharded over the ranks of `comm` (all-gather of the
    iterate per operator application).  Returns (samples, sample_tri, p (n_sys, M), infos)."""
    pr = _prec(prec)
    dev = mesh.vxyz.device
    g_tri = torch.atleast_2d(g_tri).to(torch.complex128).contiguous()
    ks, kp = _karr(k)
    n_sys = ks.size
    if out is None:
        smp = torch.empty(6, M, dtype=torch.float64, device=dev)
        tri = torch.empty(M, dtype=torch.int32, device=dev)
        p = torch.empty(n_sys, M, dtype=torch.complex128, device=dev)
    else:
        smp, tri, p = out
    world = comm.world if comm else 1
    if ws is None:
        ws = _ws(lib().nat_mc_sharded_workspace(pr, M, n_sys, max_iter, world), dev)
    opts = _McOpts(M, seed, stream_id, float(eps), _ptr(samples_in), _ptr(sample_tri_in))
    infos = (_SolveInfo * n_sys)()
    st = lib().nat_mc_surface_pressure_sharded(comm.handle if comm else None, C.byref(mesh.c()), C.byref(geom.c()),
                                               n_sys, kp, _ptr(g_tri), C.byref(opts), pr, float(tol), int(max_iter),
                                               _ptr(smp), _ptr(tri), _ptr(p), _ptr(ws), ws.numel(), infos, _stream())
    _check(st, allow_warn=True)
    return smp, tri, p, [dict(iters=i.iters, converged=i.converged, rel_residual=i.rel_residual,
                              t_total_s=i.t_total_s, t_matvec_s=i.t_matvec_s) for i in infos]


def row_range(n: int, rank: int, world: int):
    """Row ownership of the row-sharded solve: ceil(n/world) rows per rank."""
    rpr = -(-n // world)
    return min(n, rank * rpr), min(n, (rank + 1) * rpr)


def nat_bem_solve(A_local: torch.Tensor, b_local: torch.Tensor, n: int, row_begin=0, comm: Optional[Comm] = None,
                  tol=1e-6, max_iter=200, ws=None, out=None):
    """Returns (x c128 [n], info dict).  Raises on errors; non-convergence is reported
    in info['converged'] (status NAT_WARN_NOT_CONVERGED)."""
    pr = NAT_FP32 if A_local.dtype == torch.complex64 else NAT_FP64
    rows, lda = A_local.shape
    dev = A_local.device
    x = torch.empty(n, dtype=torch.complex128, device=dev) if out is None else out
    if ws is None:
        ws = _ws(lib().nat_bem_solve_workspace(pr, n, rows, max_iter), dev)
    info = _SolveInfo()
    st = lib().nat_bem_solve(comm.handle if comm else None, pr, n, row_begin, row_begin + rows, _ptr(A_local),
                             lda, _ptr(b_local.contiguous()), _ptr(x), float(tol), int(max_iter), _ptr(ws),
                             ws.numel(), C.byref(info), _stream())
    _check(st, allow_warn=True)
    return x, dict(iters=info.iters, converged=info.converged, rel_residual=info.rel_residual,
                   t_total_s=info.t_total_s, t_matvec_s=info.t_matvec_s, t_comm_s=info.t_comm_s)


# ------------------------------------------------------------------------------------
# NEXT-3: matrix-free dense operator (include/nat.h, nat_bem_mf_*)
# ------------------------------------------------------------------------------------
class BemMf:
    """The matrix-free operator of rows [near.row_begin, near.row_end): keeps the C
    structs alive and owns the near / diagonal corrections (c128 tensors)."""

    def __init__(self, mesh: Mesh, geom: Geom, near: NearList, k: float, prec="fp32", opts=None):
        self.mesh, self.geom, self.near = mesh, geom, near
        self.prec = _prec(prec)
        self.k = float(k)
        dev = mesh.vxyz.device
        rows = near.row_end - near.row_begin
        self.delta = torch.zeros(max(near.nnz, 1), dtype=torch.complex128, device=dev)
        self.diag = torch.zeros(rows, dtype=torch.complex128, device=dev)
        self._m = mesh.c()
        self._g = geom.c()
        self._o = opts or quad_opts()
        self.c = _BemMf(C.pointer(self._m), C.pointer(self._g), C.pointer(self._o), self.k, self.prec,
                        near.row_begin, near.row_end, _ptr(near.row_ptr), C.c_void_p(near.col.data_ptr()),
                        C.c_void_p(near.cls.data_ptr()), int(near.nnz), _ptr(self.delta), _ptr(self.diag))
        self._ws = None

    @property
    def rows(self):
        return self.near.row_end - self.near.row_begin

    def ws(self, n_rhs=0):
        need = lib().nat_bem_mf_workspace(C.byref(self.c), self.near.nnz, n_rhs)
        if self._ws is None or self._ws.numel() < need:
            self._ws = _ws(need, self.mesh.vxyz.device)
        return self._ws


def nat_bem_mf_prepare(mesh: Mesh, geom: Geom, near: NearList, k: float, g=None, prec="fp32", opts=None):
    """Builds the matrix-free operator (near / diagonal corrections) and rhs = -V g.
    Returns (BemMf, rhs c128 [n_rhs][rows] or None)."""
    op = BemMf(mesh, geom, near, k, prec, opts)
    n_rhs, rhs = 0, None
    if g is not None:
        g = torch.atleast_2d(g).to(torch.complex128).contiguous()
        n_rhs = g.shape[0]
        rhs = torch.empty(n_rhs, op.rows, dtype=torch.complex128, device=mesh.vxyz.device)
    ws = op.ws(n_rhs)
    _check(lib().nat_bem_mf_prepare(C.byref(op.c), n_rhs, _ptr(g), _ptr(rhs), _ptr(ws), ws.numel(), _stream()))
    return op, rhs


def nat_bem_mf_matvec(op: BemMf, x: torch.Tensor, out=None):
    """y = A x on the operator's rows (A re-evaluated, never stored)."""
    out = torch.empty(op.rows, dtype=torch.complex128, device=x.device) if out is None else out
    ws = op.ws()
    _check(lib().nat_bem_mf_matvec(C.byref(op.c), _ptr(x.to(torch.complex128).contiguous()), _ptr(out), _ptr(ws),
                                   ws.numel(), _stream()))
    return out


def nat_bem_mf_solve(op: BemMf, b_local: torch.Tensor, comm: Optional["Comm"] = None, tol=1e-6, max_iter=200,
                     out=None):
    """GMRES over the matrix-free operator (row-sharded like nat_bem_solve).
    Returns (x c128 [n], info dict)."""
    n = op.mesh.n_tri
    dev = b_local.device
    x = torch.empty(n, dtype=torch.complex128, device=dev) if out is None else out
    world = comm.world if comm else 1
    ws = _ws(lib().nat_bem_mf_solve_workspace(C.byref(op.c), max_iter, world), dev)
    info = _SolveInfo()
    st = lib().nat_bem_mf_solve(comm.handle if comm else None, C.byref(op.c), _ptr(b_local.contiguous()), _ptr(x),
                                float(tol), int(max_iter), _ptr(ws), ws.numel(), C.byref(info), _stream())
    _check(st, allow_warn=True)
    return x, dict(iters=info.iters, converged=info.converged, rel_residual=info.rel_residual,
                   t_total_s=info.t_total_s, t_matvec_s=info.t_matvec_s, t_comm_s=info.t_comm_s)


# ------------------------------------------------------------------------------------
# diagnostics: per-kernel CUDA-event timer (nat_kernel_timer_*)
# ------------------------------------------------------------------------------------
KTIMER_MC_OP, KTIMER_MC_RHS, KTIMER_RADIATE, KTIMER_FAR, KTIMER_NF_GEMM = 0, 1, 2, 3, 4


def nat_krylov_config(cluster_ctas: int, threads: int, smem_cap_kb: int):
    """Process-wide shape of the fused Arnoldi step (include/nat.h)."""
    _check(lib().nat_krylov_config(int(cluster_ctas), int(threads), int(smem_cap_kb)))


def nat_mc_set_groups(groups: int):
    """Process-wide solve groups of nat_mc_surface_pressure (include/nat.h)."""
    _check(lib().nat_mc_set_groups(int(groups)))


def nat_kernel_timer_enable(on: bool = True):
    lib().nat_kernel_timer_enable(int(bool(on)))


def nat_kernel_timer_read(category: int, n_modes: int = 0):
    """(seconds, pair-evaluations x wavenumbers, launches) of the category's main kernel
    since enable; n_modes > 0: only the launches with that many wavenumbers per pair."""
    sec, pairs, n = C.c_double(0.0), C.c_double(0.0), C.c_int64(0)
    _check(lib().nat_kernel_timer_read_modes(int(category), int(n_modes), C.byref(sec), C.byref(pairs), C.byref(n)))
    return sec.value, pairs.value, n.value


# ------------------------------------------------------------------------------------
# NEXT-4: the NAT neural field (include/nat.h, nat_nf_*)
# ------------------------------------------------------------------------------------
class NeuralField:
    """Parameters (fp32, device), Adam moments and a workspace for batches of up to
    `max_batch` samples.  Inputs [n][3 + n_v] (normalised theta, phi, r, conditions),
    outputs [n][n_out]."""

    def __init__(self, n_v: int, n_out: int, params: torch.Tensor, max_batch: int):
        self.cfg = _NfConfig(int(n_v), int(n_out))
        n = lib().nat_nf_param_count(C.byref(self.cfg))
        if n < 0:
            raise NatError(-1, f"bad neural-field config n_v = {n_v}, n_out = {n_out}")
        if params.numel() != n:
            raise NatError(-1, f"{params.numel()} parameters, the layout has {n}")
        self.params = params.to(torch.float32).contiguous()
        self.m = torch.zeros_like(self.params)
        self.v = torch.zeros_like(self.params)
        self.step = 0
        self.max_batch = int(max_batch)
        self.ws = _ws(lib().nat_nf_workspace(C.byref(self.cfg), self.max_batch), self.params.device)
        self.loss = torch.zeros(1, dtype=torch.float32, device=self.params.device)

    @staticmethod
    def param_count(n_v: int, n_out: int) -> int:
        return int(lib().nat_nf_param_count(C.byref(_NfConfig(int(n_v), int(n_out)))))

    @staticmethod
    def param_shapes(n_v: int, n_out: int):
        """Block shapes of the parameter vector as include/nat.h documents it: 4 lattices
        [(N+1)^3][4], N = 8, 16, 32, 64, then W [out][in] and b [out] of the 5 layers."""
        shapes = [((8 << l) + 1) ** 3 for l in range(4)]
        shapes = [(min(r, 1 << 19), 4) for r in shapes]
        dims = [64, 128, 128, 128, 128, int(n_out)]
        for q in range(5):
            shapes += [(dims[q + 1], dims[q]), (dims[q + 1],)]
        if sum(int(np.prod(s)) for s in shapes) != NeuralField.param_count(n_v, n_out):
            raise NatError(-1, "parameter layout mismatch with libnat")
        return shapes

    def forward(self, inputs: torch.Tensor, out=None):
        n = inputs.shape[0]
        out = torch.empty(n, self.cfg.n_out, dtype=torch.float32, device=inputs.device) if out is None else out
        _check(lib().nat_nf_forward(C.byref(self.cfg), _ptr(self.params), n, _ptr(inputs), _ptr(out), _ptr(self.ws),
                                    self.ws.numel(), _stream()))
        return out

    def train_step(self, inputs: torch.Tensor, targets: torch.Tensor, lr: float, grad_out=None):
        """One forward / MSE / backward / Adam step; returns the loss tensor (device, before
        the update)."""
        self.step += 1
        _check(lib().nat_nf_train_step(C.byref(self.cfg), _ptr(self.params), _ptr(self.m), _ptr(self.v), self.step,
                                       float(lr), inputs.shape[0], _ptr(inputs), _ptr(targets), _ptr(self.loss),
                                       _ptr(grad_out), _ptr(self.ws), self.ws.numel(), _stream()))
        return self.loss


def nat_nf_gemm_bf16(A: torch.Tensor, B: torch.Tensor, a_mn=False, b_mn=False, out=None):
    """C = A B^T on the tcgen05 tensor cores: A bf16 [M][K] (or [K][M] with a_mn), B bf16
    [N][K] (or [K][N] with b_mn); returns fp32 [M][N]."""
    M = A.shape[1] if a_mn else A.shape[0]
    K = A.shape[0] if a_mn else A.shape[1]
    N = B.shape[1] if b_mn else B.shape[0]
    out = torch.empty(M, N, dtype=torch.float32, device=A.device) if out is None else out
    _check(lib().nat_nf_gemm_bf16(M, N, K, _ptr(A), A.shape[1], int(bool(a_mn)), _ptr(B), B.shape[1],
                                  int(bool(b_mn)), _ptr(out), out.shape[1], _stream()))
    return out
