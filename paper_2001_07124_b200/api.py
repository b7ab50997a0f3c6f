"""Thin Python binding of librtucker with the C-ABI's names (argument marshalling only).

Every step of the hot path runs in the library's CUDA kernels; torch provides the
device buffers and the stream.  Conventions:

  * a tensor X with math shape (I_1, ..., I_N) is a C-contiguous torch tensor of shape
    (I_N, ..., I_1) (first-mode-fastest memory, gen.synth.to_device_layout);
  * an m x k "col-major" matrix is a torch tensor M of shape (m, k) with strides (1, m)
    (i.e. ``t.T`` of a contiguous (k, m) tensor); results are returned that way;
  * Gaussian Omega_n (J_n, K_n) and Kronecker factors (d_k, L_k) are passed to the library
    column-major; any (rows, cols) torch tensor is accepted (a strided column-major view such as
    a slab's row block Omega[r0:r1, :] of a column-major Omega is used in place, otherwise a
    column-major copy is made).
"""
from __future__ import annotations

import ctypes as C
import math
from typing import List, Optional, Sequence

import torch

from . import _lib as L
from ._lib import RtError, lib


def _check(h, st: int):
    if st != 0:
        msg = lib.rt_last_error(h.ptr if h is not None else None)
        raise RtError(st, (msg or b"").decode(errors="replace"))


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return L.RT_F32
    if t.dtype == torch.float64:
        return L.RT_F64
    raise TypeError(f"unsupported dtype {t.dtype}")


def colmajor(m: torch.Tensor) -> torch.Tensor:
    """(m, k) tensor with col-major storage (strides (1, m))."""
    if m.dim() != 2:
        raise ValueError("expected a matrix")
    if m.stride(0) == 1 and (m.stride(1) == m.shape[0] or m.shape[1] == 1):
        return m
    return m.t().contiguous().t()


def colmajor_ld(m: torch.Tensor):
    """(tensor, ld): a column-major view (stride(0) == 1, stride(1) = ld >= rows) used in place,
    else a packed column-major copy."""
    if m.dim() != 2:
        raise ValueError("expected a matrix")
    if m.stride(0) == 1 and m.stride(1) >= m.shape[0]:
        return m, (m.stride(1) if m.shape[1] > 1 else max(1, m.shape[0]))
    c = m.t().contiguous().t()
    return c, max(1, c.shape[0])


def rowmajor_ld(m: torch.Tensor):
    """(tensor, ld): a row-major view (stride(1) == 1, stride(0) = ld >= cols) used in place, else a
    packed row-major copy (the layout of every test matrix Omega, include/rtucker.h)."""
    if m.dim() != 2:
        raise ValueError("expected a matrix")
    if m.stride(1) == 1 and m.stride(0) >= m.shape[1]:
        return m, (m.stride(0) if m.shape[0] > 1 else max(1, m.shape[1]))
    c = m.contiguous()
    return c, max(1, c.shape[1])


def new_colmajor(m: int, k: int, dtype=torch.float64, device=None) -> torch.Tensor:
    return torch.empty((k, m), dtype=dtype, device=device).t()


class Handle:
    """rt_handle: stream + optional communicator + workspace."""

    def __init__(self, stream: Optional[torch.cuda.Stream] = None, nccl_id: Optional[bytes] = None,
                 nranks: int = 1, rank: int = 0, loopback_group: "Optional[LoopbackGroup]" = None):
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        self.ptr = C.c_void_p()
        self.rank, self.nranks = rank, nranks
        self._keep: list = []
        if loopback_group is not None:
            st = lib.rt_create_loopback(C.byref(self.ptr), C.c_void_p(self.stream.cuda_stream),
                                        loopback_group.ptr, rank)
            self.nranks = loopback_group.nranks
        else:
            idbuf = None
            if nccl_id is not None:
                idbuf = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
            st = lib.rt_create(C.byref(self.ptr), C.c_void_p(self.stream.cuda_stream), idbuf, nranks, rank)
        if st != 0:
            raise RtError(st, (lib.rt_last_error(None) or b"").decode())

    def keep(self, *objs):
        self._keep.extend(objs)

    def sync(self):
        st = lib.rt_sync(self.ptr)
        self._keep.clear()
        _check(self, st)

    def set_option(self, opt: int, value: int):
        _check(self, lib.rt_set_option(self.ptr, opt, int(value)))

    def profile_read(self):
        cap = 64
        buf = (L.rt_profile_entry * cap)()
        n = C.c_int(0)
        launches = C.c_int64(0)
        _check(self, lib.rt_profile_read(self.ptr, buf, cap, C.byref(n), C.byref(launches)))
        return [(buf[i].name.decode(), int(buf[i].count), float(buf[i].ms)) for i in range(n.value)], int(launches.value)

    def close(self):
        if self.ptr:
            lib.rt_destroy(self.ptr)
            self.ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LoopbackGroup:
    """In-process communicator group for emulating ranks on one GPU (one host thread per rank)."""

    def __init__(self, nranks: int):
        self.ptr = C.c_void_p()
        self.nranks = nranks
        st = lib.rt_loopback_group_create(C.byref(self.ptr), nranks)
        if st != 0:
            raise RtError(st, "loopback group")

    def __del__(self):
        if self.ptr:
            lib.rt_loopback_group_destroy(self.ptr)


def get_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    st = lib.rt_get_unique_id(buf)
    if st != 0:
        raise RtError(st, (lib.rt_last_error(None) or b"").decode())
    return bytes(buf)


def tensor_desc(x: torch.Tensor, last_offset: int = 0, last_global: Optional[int] = None) -> L.rt_tensor:
    if not x.is_cuda or not x.is_contiguous():
        raise ValueError("X must be a contiguous CUDA tensor of shape (I_N, ..., I_1)")
    dims = list(reversed(x.shape))
    if not 2 <= len(dims) <= 5:
        raise ValueError("order must be in [2, 5]")
    t = L.rt_tensor()
    t.dtype = _dtype_code(x)
    t.order = len(dims)
    for k, d in enumerate(dims):
        t.dims[k] = int(d)
    t.last_offset = int(last_offset)
    t.last_global = int(dims[-1] if last_global is None else last_global)
    t.data = x.data_ptr()
    return t


def _ptr_array(ts) -> "C.Array":
    arr = (C.c_void_p * len(ts))()
    for i, t in enumerate(ts):
        arr[i] = None if t is None else t.data_ptr()
    return arr


def _i64_array(vals) -> "C.Array":
    arr = (C.c_int64 * len(vals))()
    for i, v in enumerate(vals):
        arr[i] = int(v)
    return arr


def _omega_table(N: int, omegas, kind: str):
    """Flat N x N tables (pointer, cols, ld) indexed [n*N + k] (include/rtucker.h)."""
    ptrs = [None] * (N * N)
    cols = [0] * (N * N)
    lds = [0] * (N * N)
    keep = []
    for n in range(N):
        if kind == "count":
            codes, K = _count_codes(omegas[n])
            keep.append(codes)
            ptrs[n * N + n], cols[n * N + n], lds[n * N + n] = codes, K, 1
            continue
        entries = [(n, omegas[n])] if kind == "gauss" else \
            [(k, omegas[n][k]) for k in range(N) if k != n and omegas[n][k] is not None]
        for k, om in entries:
            om, ld = rowmajor_ld(om)
            keep.append(om)
            ptrs[n * N + k] = om
            cols[n * N + k] = om.shape[1]
            lds[n * N + k] = ld
    return _ptr_array(ptrs), _i64_array(cols), _i64_array(lds), keep


def _kind(kind: str) -> int:
    return {"gauss": L.RT_OMEGA_GAUSS, "kron": L.RT_OMEGA_KRON, "kr": L.RT_OMEGA_KR,
            "count": L.RT_OMEGA_COUNT}[kind]


def _count_codes(entry):
    """Count-sketch operand (codes, K): codes = int32 device vector, code_j = s_j (h_j + 1)."""
    codes, K = entry
    if codes.dtype != torch.int32 or codes.dim() != 1:
        raise ValueError("count-sketch codes must be a 1-D int32 tensor")
    return codes.contiguous(), int(K)


def rtucker_sketch(h: Handle, X: torch.Tensor, mode: int, omega, q: int = 0, kind: str = "gauss",
                   last_offset: int = 0, last_global: Optional[int] = None) -> torch.Tensor:
    """Y = X_(n) Omega (+ q power iterations); returns fp64 (I_n_local, K) col-major."""
    desc = tensor_desc(X, last_offset, last_global)
    N = desc.order
    ptrs, cols, lds, keep = [None] * N, [0] * N, [0] * N, []
    if kind == "count":
        codes, K = _count_codes(omega)
        keep.append(codes)
        if 0 <= mode < N:
            ptrs[mode], cols[mode], lds[mode] = codes, K, 1
    elif kind == "gauss":
        om, ld = rowmajor_ld(omega)
        keep.append(om)
        K = om.shape[1]
        if 0 <= mode < N:              # out-of-range modes are rejected by the library (RT_EINVAL)
            ptrs[mode], cols[mode], lds[mode] = om, K, ld
    else:
        K = 1
        for k in range(N):
            if k == mode:
                continue
            o, ld = rowmajor_ld(omega[k])
            keep.append(o)
            ptrs[k], cols[k], lds[k] = o, o.shape[1], ld
            K = o.shape[1] if kind == "kr" else K * o.shape[1]     # Khatri-Rao: shared width
    In = desc.dims[mode] if 0 <= mode < N else 1
    Y = new_colmajor(In, K, device=X.device)
    st = lib.rtucker_sketch(h.ptr, C.byref(desc), mode, _kind(kind), _ptr_array(ptrs), _i64_array(cols),
                            _i64_array(lds), q, C.c_void_p(Y.data_ptr()), In)
    h.keep(*keep)
    _check(h, st)
    return Y


def rtucker_qr(h: Handle, Y: torch.Tensor, rows_distributed: bool = False):
    """Thin QR Y = QR (R_ii >= 0); returns (Q fp64 col-major (m, k), R fp64 (k, k))."""
    Yc = colmajor(Y)
    m, k = Yc.shape
    Q = new_colmajor(m, k, device=Y.device)
    R = new_colmajor(k, k, device=Y.device)
    st = lib.rtucker_qr(h.ptr, m, k, _dtype_code(Yc), C.c_void_p(Yc.data_ptr()), max(m, 1),
                        C.c_void_p(Q.data_ptr()), max(m, 1), C.c_void_p(R.data_ptr()), int(rows_distributed))
    h.keep(Yc)
    _check(h, st)
    return Q, R


def rtucker_core(h: Handle, X: torch.Tensor, Qs: Sequence[torch.Tensor], with_error: bool = True,
                 last_offset: int = 0, last_global: Optional[int] = None):
    """G = X x_n Q_n^T (all n) and optionally (E, E_gram).  Returns (G, err) with G of device
    layout (C_N, ..., C_1) and err a fp64 device tensor [E, E_gram] (or None)."""
    desc = tensor_desc(X, last_offset, last_global)
    Qc = [colmajor(q.to(torch.float64)) for q in Qs]
    Cs = [q.shape[1] for q in Qc]
    G = torch.empty(tuple(reversed(Cs)), dtype=torch.float64, device=X.device)
    err = torch.zeros(2, dtype=torch.float64, device=X.device) if with_error else None
    st = lib.rtucker_core(h.ptr, C.byref(desc), _ptr_array(Qc), _i64_array(Cs), C.c_void_p(G.data_ptr()),
                          C.c_void_p(err.data_ptr()) if with_error else None,
                          C.c_void_p(err.data_ptr() + 8) if with_error else None)
    h.keep(*Qc)
    _check(h, st)
    return G, err


def _driver(fn, h, X, ranks, p, q, omegas, kind, with_error, last_offset, last_global, mode_order=None):
    desc = tensor_desc(X, last_offset, last_global)
    N = desc.order
    ptrs, cols, lds, keep = _omega_table(N, omegas, kind)
    local = [desc.dims[n] for n in range(N)]
    Q = [new_colmajor(local[n], ranks[n], device=X.device) for n in range(N)]
    G = torch.empty(tuple(reversed(list(ranks))), dtype=torch.float64, device=X.device)
    err = torch.zeros(2, dtype=torch.float64, device=X.device) if with_error else None
    args = [h.ptr, C.byref(desc), _i64_array(ranks), int(p), int(q), _kind(kind), ptrs, cols, lds]
    if fn is lib.rtucker_sthosvd:
        if mode_order is None:
            args.append(None)
        else:
            mo = (C.c_int * N)(*[int(m) for m in mode_order])
            args.append(mo)
    args += [_ptr_array(Q), C.c_void_p(G.data_ptr()),
             C.c_void_p(err.data_ptr()) if with_error else None,
             C.c_void_p(err.data_ptr() + 8) if with_error else None]
    st = fn(*args)
    h.keep(*keep)
    _check(h, st)
    return dict(Q=Q, G=G, err=err)


def rtucker_hosvd(h: Handle, X: torch.Tensor, ranks: Sequence[int], p: int, q: int, omegas, kind: str = "gauss",
                  with_error: bool = True, last_offset: int = 0, last_global: Optional[int] = None) -> dict:
    """Randomized HOSVD (Alg.6 + Alg.1 oversampling/power iteration + R1 truncation).
    Returns dict(Q=[fp64 (I_n_local, R_n) col-major], G=fp64 device-layout core, err=[E, E_gram])."""
    return _driver(lib.rtucker_hosvd, h, X, ranks, p, q, omegas, kind, with_error, last_offset, last_global)


def rtucker_sthosvd(h: Handle, X: torch.Tensor, ranks: Sequence[int], p: int, q: int, omegas, kind: str = "gauss",
                    mode_order: Optional[Sequence[int]] = None, with_error: bool = True, last_offset: int = 0,
                    last_global: Optional[int] = None) -> dict:
    """Randomized STHOSVD (Alg.8).  omegas sized for the shrinking working tensor (local rows of
    the slab for modes processed before the slab mode, which must come last when sharded)."""
    return _driver(lib.rtucker_sthosvd, h, X, ranks, p, q, omegas, kind, with_error, last_offset, last_global,
                   mode_order)


def rtucker_pet(h: Handle, X: torch.Tensor, ranks: Sequence[int], omegas, omega_tildes, with_error: bool = True,
                last_offset: int = 0, last_global: Optional[int] = None) -> dict:
    """Randomized pass-efficient Tucker (Alg.9 R-PET).  omegas[n]: Omega_n (J_n x K_n);
    omega_tildes[n]: Omega~_n (S_n x I_n, local columns of the last mode on a slab).
    Returns dict(Q, G, err) as rtucker_hosvd."""
    desc = tensor_desc(X, last_offset, last_global)
    N = desc.order
    ptrs, cols, lds, keep = _omega_table(N, omegas, "gauss")
    tl, tp, tld = [], [], []
    for o in omega_tildes:
        o, ld = rowmajor_ld(o)
        tl.append(o)
        tp.append(o)
        tld.append(ld)
    S = [int(o.shape[0]) for o in tl]
    local = [desc.dims[n] for n in range(N)]
    Q = [new_colmajor(local[n], ranks[n], device=X.device) for n in range(N)]
    G = torch.empty(tuple(reversed(list(ranks))), dtype=torch.float64, device=X.device)
    err = torch.zeros(2, dtype=torch.float64, device=X.device) if with_error else None
    st = lib.rtucker_pet(h.ptr, C.byref(desc), _i64_array(ranks), ptrs, cols, lds, _ptr_array(tp), _i64_array(S),
                         _i64_array(tld), _ptr_array(Q), C.c_void_p(G.data_ptr()),
                         C.c_void_p(err.data_ptr()) if with_error else None,
                         C.c_void_p(err.data_ptr() + 8) if with_error else None)
    h.keep(*keep, *tl)
    _check(h, st)
    return dict(Q=Q, G=G, err=err)


def rtucker_rp_hooi(h: Handle, X: torch.Tensor, ranks: Sequence[int], q_init, omegas, with_error: bool = True,
                    last_offset: int = 0, last_global: Optional[int] = None) -> dict:
    """Random projection HOOI (Alg.7).  q_init[n]: fp64 (I_n_local, R_n) starting factors;
    omegas[sweep][n]: fp64 (prod_{p!=n} R_p, R_n).  Returns dict(Q, G, err) as rtucker_hosvd."""
    desc = tensor_desc(X, last_offset, last_global)
    N = desc.order
    q0 = [colmajor(q.to(torch.float64)) for q in q_init]
    for n, q in enumerate(q0):
        if q.stride(1) != q.shape[0] and q.shape[1] > 1:
            raise ValueError("q_init must be packed column-major")
    flat, lds, keep = [], [], list(q0)
    for sweep in omegas:
        if len(sweep) != N:
            raise ValueError("each sweep needs N test matrices")
        for n, o in enumerate(sweep):
            rows = math.prod(int(ranks[p]) for p in range(N) if p != n)
            if tuple(o.shape) != (rows, ranks[n]):
                raise ValueError(f"Omega^({n}) must be ({rows}, {ranks[n]}), got {tuple(o.shape)}")
            o, ld = rowmajor_ld(o.to(torch.float64))
            keep.append(o)
            flat.append(o)
            lds.append(ld)
    local = [desc.dims[n] for n in range(N)]
    Q = [new_colmajor(local[n], ranks[n], device=X.device) for n in range(N)]
    G = torch.empty(tuple(reversed(list(ranks))), dtype=torch.float64, device=X.device)
    err = torch.zeros(2, dtype=torch.float64, device=X.device) if with_error else None
    st = lib.rtucker_rp_hooi(h.ptr, C.byref(desc), _i64_array(ranks), len(omegas), _ptr_array(q0),
                             _ptr_array(flat) if flat else None, _i64_array(lds) if lds else None, _ptr_array(Q),
                             C.c_void_p(G.data_ptr()), C.c_void_p(err.data_ptr()) if with_error else None,
                             C.c_void_p(err.data_ptr() + 8) if with_error else None)
    h.keep(*keep)
    _check(h, st)
    return dict(Q=Q, G=G, err=err)


def core_to_numpy(G: torch.Tensor):
    """Device-layout core (R_N..R_1) -> numpy array indexed G[r_1, ..., r_N]."""
    return G.detach().cpu().numpy().T


__all__ = ["Handle", "LoopbackGroup", "get_unique_id", "tensor_desc", "colmajor", "new_colmajor",
           "rtucker_sketch", "rtucker_qr", "rtucker_core", "rtucker_hosvd", "rtucker_sthosvd", "core_to_numpy",
           "RtError"]
