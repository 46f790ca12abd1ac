"""Thin Python binding of libsfairsc (include/sfairsc.h) — argument marshalling only.

Every step of the s-FairSC path runs in the CUDA library; this module only
converts numpy arrays / torch tensors to pointers, calls the C ABI and raises
`SfairscError` on a non-OK status.  There is no CPU fallback: if the shared
library is missing or fails to load, importing this module raises.

Names mirror the C ABI: sfairsc_build_operator, sfairsc_eigs,
sfairsc_embed_kmeans, sfairsc_apply, sfairsc_project, sfairsc_laplacian, ...
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libsfairsc.so")

MEM_HOST = 0
MEM_DEVICE = 1

STATUS = {
    0: "OK", 1: "E_INVALID_ARG", 2: "E_DIM_MISMATCH", 3: "E_CSR_INVALID", 4: "E_ASYMMETRIC",
    5: "E_NEGATIVE_WEIGHT", 6: "E_ISOLATED_VERTEX", 7: "E_EMPTY_GROUP", 8: "E_RANK_DEFICIENT",
    9: "E_K_TOO_LARGE", 10: "E_SHIFT_TOO_SMALL", 11: "E_NO_CONVERGENCE", 12: "E_STATE", 13: "E_OOM",
    14: "E_CUDA", 15: "E_NCCL",
}

PROFILE_KINDS = {"spmv": 0, "dots": 1, "upd_dots": 2, "upd_norm": 3, "normalize": 4, "ritz": 5,
                 "project": 6, "finish": 7, "kmeans": 8, "other": 9}


class SfairscError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__(f"{self.name}: {msg}")


class CSR(C.Structure):
    _fields_ = [("n_rows", C.c_int64), ("n_cols", C.c_int64), ("nnz", C.c_int64), ("row_offset", C.c_int64),
                ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p), ("values", C.c_void_p), ("memspace", C.c_int32)]


class Opts(C.Structure):
    _fields_ = [("sigma_override", C.c_double), ("max_basis", C.c_int32), ("keep", C.c_int32),
                ("max_restarts", C.c_int32), ("start_seed", C.c_uint64), ("tol_eff_cap", C.c_double),
                ("cuda_stream", C.c_void_p), ("check_symmetry", C.c_int32), ("spmv_vector", C.c_int32),
                ("block_size", C.c_int32), ("reorth", C.c_int32), ("comm", C.c_void_p),
                ("virtual_parts", C.c_int32), ("filter_degree", C.c_int32), ("filter_cut", C.c_double)]


class Stats(C.Structure):
    _fields_ = [("applies", C.c_int64), ("steps", C.c_int64), ("restarts", C.c_int64), ("breakdowns", C.c_int64),
                ("sigma", C.c_double), ("max_resid_rel", C.c_double), ("gap_est", C.c_double),
                ("t_build_s", C.c_double), ("t_eigs_s", C.c_double), ("converged", C.c_int32),
                ("basis_size", C.c_int32), ("kept", C.c_int32), ("reserved", C.c_int32),
                ("filter_cut", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_ if f != "reserved"}


class Info(C.Structure):
    _fields_ = [("n", C.c_int64), ("nnz", C.c_int64), ("h", C.c_int32), ("k_build", C.c_int32),
                ("normalized", C.c_int32), ("spmv_vector", C.c_int32), ("sigma", C.c_double),
                ("device", C.c_int32), ("num_sms", C.c_int32), ("unit_weights", C.c_int32),
                ("constraint_rank", C.c_int32)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libsfairsc.so not built at {LIB_PATH}; run `python -m paper_2210_16435_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P = C.c_void_p
    sig = {
        "sfairsc_default_opts": (None, [C.POINTER(Opts)]),
        "sfairsc_build_operator": (C.c_int, [C.POINTER(CSR), P, C.c_int32, C.c_int32, C.c_int32, C.POINTER(P)]),
        "sfairsc_build_operator_ex": (C.c_int, [C.POINTER(CSR), P, C.c_int32, C.c_int32, C.c_int32,
                                                C.POINTER(Opts), C.POINTER(P)]),
        "sfairsc_eigs": (C.c_int, [P, C.c_int32, C.c_double, P, P, C.c_int32, C.POINTER(Stats)]),
        "sfairsc_embed_kmeans": (C.c_int, [P, C.c_uint64, P, C.c_int32, P]),
        "sfairsc_apply": (C.c_int, [P, P, P, C.c_int32, C.c_int32]),
        "sfairsc_apply_ex": (C.c_int, [P, P, P, C.c_int32, C.c_int32, C.c_int32]),
        "sfairsc_project": (C.c_int, [P, P, P, C.c_int32, C.c_int32]),
        "sfairsc_laplacian": (C.c_int, [P, P, P, C.c_int32]),
        "sfairsc_get_info": (C.c_int, [P, C.POINTER(Info)]),
        "sfairsc_profile_enable": (C.c_int, [P, C.c_int32]),
        "sfairsc_profile_read": (C.c_int, [P, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                           C.POINTER(C.c_double)]),
        "sfairsc_launch_count": (C.c_int64, []),
        "sfairsc_profile_reset": (C.c_int, [P]),
        "sfairsc_destroy": (None, [P]),
        "sfairsc_last_error": (C.c_char_p, []),
        "sfairsc_version": (C.c_char_p, []),
        "sfairsc_host_symeig": (C.c_int, [C.c_int32, P, P, P]),
        "sfairsc_host_symeig_sel": (C.c_int, [C.c_int32, P, P, P, C.c_int32]),
        "sfairsc_build_operator_dense": (C.c_int, [C.POINTER(CSR), P, C.c_int32, C.c_int32, C.c_int32,
                                                   C.POINTER(Opts), C.POINTER(P)]),
        "sfairsc_comm_unique_id": (C.c_int, [P]),
        "sfairsc_comm_init": (C.c_int, [P, C.c_int32, C.c_int32, C.c_int32, C.POINTER(P)]),
        "sfairsc_comm_destroy": (None, [P]),
        "sfairsc_struct_size": (C.c_int64, [C.c_int32]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    # the struct mirrors above must match the library's layout (include/sfairsc.h)
    for which, st in enumerate((CSR, Opts, Stats, Info)):
        if lib.sfairsc_struct_size(which) != C.sizeof(st):
            raise ImportError(f"{st.__name__}: ctypes size {C.sizeof(st)} != library {lib.sfairsc_struct_size(which)}"
                              " (stale build of libsfairsc.so?)")
    return lib


_lib = _load()


def version() -> str:
    return _lib.sfairsc_version().decode()


def _check(status: int):
    if status != 0:
        raise SfairscError(status, _lib.sfairsc_last_error().decode())


def _is_torch(x):
    return type(x).__module__.startswith("torch")


def _ptr(x, dtype):
    """(pointer, memspace) of a contiguous numpy array or torch tensor of `dtype`."""
    if _is_torch(x):
        import torch
        tdt = {np.float64: torch.float64, np.int32: torch.int32}[dtype]
        if x.dtype != tdt or not x.is_contiguous():
            raise TypeError(f"expected contiguous {tdt} tensor")
        return x.data_ptr(), (MEM_DEVICE if x.is_cuda else MEM_HOST)
    if not isinstance(x, np.ndarray) or x.dtype != dtype or not x.flags.c_contiguous:
        raise TypeError(f"expected C-contiguous numpy {np.dtype(dtype)} array")
    return x.ctypes.data, MEM_HOST


def default_opts(**kw) -> Opts:
    o = Opts()
    _lib.sfairsc_default_opts(C.byref(o))
    for k, v in kw.items():
        if k == "cuda_stream" and v is not None and not isinstance(v, int):
            v = v.cuda_stream  # torch.cuda.Stream
        if k == "comm" and isinstance(v, Comm):
            v = v.handle.value
        setattr(o, k, v)
    return o


class Context:
    """Owns one sfairsc_ctx (library-owned device memory)."""

    def __init__(self, handle, n: int, k: int):
        self._h = C.c_void_p(handle)
        self.n = n
        self.k = k
        self.last_stats: dict | None = None

    @property
    def handle(self):
        return self._h

    def info(self) -> dict:
        i = Info()
        _check(_lib.sfairsc_get_info(self._h, C.byref(i)))
        return {f: getattr(i, f) for f, _ in i._fields_}

    def close(self):
        if self._h:
            _lib.sfairsc_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def sfairsc_build_operator(row_ptr, col_idx, values, groups, k: int, normalized: bool, h: int = 0,
                           opts: Opts | None = None, n_global: int | None = None, row_offset: int = 0,
                           **opt_kw) -> Context:
    """Build the operator from CSR arrays (numpy host arrays or CUDA tensors;
    all four in the same memspace).  See include/sfairsc.h."""
    rp, ms = _ptr(row_ptr, np.int32)
    ci, ms2 = _ptr(col_idx, np.int32)
    vv, ms3 = _ptr(values, np.float64)
    gp, ms4 = _ptr(groups, np.int32)
    if len({ms, ms2, ms3, ms4}) != 1:
        raise ValueError("row_ptr, col_idx, values and groups must share one memspace")
    n = len(row_ptr) - 1
    nnz = len(col_idx)
    # a rank of a row-partitioned job passes its row block [row_offset, row_offset + n) of the n_global rows
    csr = CSR(n, n if n_global is None else int(n_global), nnz, int(row_offset), rp, ci, vv, ms)
    if opts is None and opt_kw:
        opts = default_opts(**opt_kw)
    out = C.c_void_p()
    if opts is None:
        _check(_lib.sfairsc_build_operator(C.byref(csr), gp, h, k, int(bool(normalized)), C.byref(out)))
    else:
        _check(_lib.sfairsc_build_operator_ex(C.byref(csr), gp, h, k, int(bool(normalized)), C.byref(opts),
                                              C.byref(out)))
    return Context(out.value, n, k)


def sfairsc_build_operator_dense(row_ptr, col_idx, values, F, k: int, normalized: bool, opts: Opts | None = None,
                                 **opt_kw) -> Context:
    """§8(f) N4: constraints C^T H = 0 with a dense F.  F: numpy (n, r) array (any order; passed
    column-major) or a CUDA tensor of shape (r, n) (= F column-major); same memspace as W."""
    rp, ms = _ptr(row_ptr, np.int32)
    ci, _ = _ptr(col_idx, np.int32)
    vv, _ = _ptr(values, np.float64)
    n = len(row_ptr) - 1
    if _is_torch(F):
        r = int(F.shape[0]) if F.ndim == 2 else 1
        fp, msf = _ptr(F.contiguous(), np.float64)
        Fk = F
    else:
        Fk = np.asfortranarray(np.asarray(F, dtype=np.float64).reshape(n, -1))
        r = Fk.shape[1]
        fp, msf = Fk.ctypes.data, MEM_HOST
    if msf != ms:
        raise ValueError("F and W must share a memspace")
    csr = CSR(n, n, len(col_idx), 0, rp, ci, vv, ms)
    if opts is None:
        opts = default_opts(**opt_kw)
    out = C.c_void_p()
    _check(_lib.sfairsc_build_operator_dense(C.byref(csr), fp if r > 0 else None, r, k, int(bool(normalized)),
                                             C.byref(opts), C.byref(out)))
    del Fk
    return Context(out.value, n, k)


def sfairsc_eigs(ctx: Context, k: int, tol: float, evecs=None, want_evecs: bool = True):
    """k smallest eigenpairs of L^sigma.  `evecs` may be a preallocated
    (k, n) C-contiguous float64 numpy array or CUDA tensor (= X^T, i.e. X
    column-major); if None and want_evecs, a numpy array is returned.
    Returns (evals ndarray, evecs (k x n) or None, stats dict)."""
    ev = np.zeros(k)
    st = Stats()
    if evecs is None and want_evecs:
        evecs = np.zeros((k, ctx.n))
    if evecs is not None:
        if tuple(evecs.shape) != (k, ctx.n):  # the library writes k x n doubles
            raise ValueError(f"evecs must have shape ({k}, {ctx.n}), got {tuple(evecs.shape)}")
        ep, ms = _ptr(evecs, np.float64)
    else:
        ep, ms = None, MEM_HOST
    status = _lib.sfairsc_eigs(ctx.handle, k, float(tol), ev.ctypes.data, ep, ms, C.byref(st))
    ctx.last_stats = st.as_dict()
    _check(status)
    return ev, evecs, ctx.last_stats


def sfairsc_embed_kmeans(ctx: Context, seed: int, labels=None):
    """Alg. 3 step 4: labels (n,) int32 (numpy or CUDA tensor) and the WCSS."""
    if labels is None:
        labels = np.zeros(ctx.n, dtype=np.int32)
    if tuple(labels.shape) != (ctx.n,):  # the library writes n int32 labels
        raise ValueError(f"labels must have shape ({ctx.n},), got {tuple(labels.shape)}")
    lp, ms = _ptr(labels, np.int32)
    obj = C.c_double()
    _check(_lib.sfairsc_embed_kmeans(ctx.handle, C.c_uint64(seed), lp, ms, C.byref(obj)))
    return labels, obj.value


def _vec_call(fn, ctx, x, y):
    xp, ms = _ptr(x, np.float64)
    if x.ndim not in (1, 2) or x.shape[-1] != ctx.n:
        raise ValueError(f"x must be (n,) or (nvec, n) with n = {ctx.n}, got {tuple(x.shape)}")
    nvec = 1 if x.ndim == 1 else x.shape[0]
    if y is None:
        if ms == MEM_DEVICE:
            import torch
            y = torch.empty_like(x)
        else:
            y = np.empty_like(x)
    if tuple(y.shape) != tuple(x.shape):
        raise ValueError(f"y must have the shape of x {tuple(x.shape)}, got {tuple(y.shape)}")
    yp, ms2 = _ptr(y, np.float64)
    if ms != ms2:
        raise ValueError("x and y must share a memspace")
    _check(fn(ctx.handle, xp, yp, nvec, ms))
    return y


def sfairsc_apply(ctx: Context, x, y=None):
    """y = L^sigma x; x is (n,) or (nvec, n) (rows = vectors)."""
    return _vec_call(_lib.sfairsc_apply, ctx, x, y)


APPLY_SINGLE = 1


def sfairsc_apply_single(ctx: Context, x, y=None):
    """y = L^sigma x one vector per SpMV (sfairsc_apply_ex with SFAIRSC_APPLY_SINGLE)."""
    return _vec_call(lambda h, xp, yp, nv, ms: _lib.sfairsc_apply_ex(h, xp, yp, nv, ms, APPLY_SINGLE), ctx, x, y)


def sfairsc_project(ctx: Context, x, y=None):
    """y = P x; x is (n,) or (nvec, n)."""
    return _vec_call(_lib.sfairsc_project, ctx, x, y)


def sfairsc_laplacian(ctx: Context, x, y=None):
    """y = L x (L_n or D - W) for one vector."""
    xp, ms = _ptr(x, np.float64)
    if y is None:
        if ms == MEM_DEVICE:
            import torch
            y = torch.empty_like(x)
        else:
            y = np.empty_like(x)
    yp, _ = _ptr(y, np.float64)
    _check(_lib.sfairsc_laplacian(ctx.handle, xp, yp, ms))
    return y


def profile_enable(ctx: Context, on: bool = True):
    _check(_lib.sfairsc_profile_enable(ctx.handle, int(on)))


def profile_reset(ctx: Context):
    _check(_lib.sfairsc_profile_reset(ctx.handle))


def profile_read(ctx: Context) -> dict:
    out = {}
    for name, kind in PROFILE_KINDS.items():
        ms = C.c_double()
        cnt = C.c_int64()
        by = C.c_double()
        _check(_lib.sfairsc_profile_read(ctx.handle, kind, C.byref(ms), C.byref(cnt), C.byref(by)))
        out[name] = {"ms": ms.value, "launches": cnt.value, "alg_bytes": by.value}
    return out


def launch_count() -> int:
    """Kernels launched by libsfairsc in this process."""
    return int(_lib.sfairsc_launch_count())


def host_symeig(A: np.ndarray):
    """Rayleigh-Ritz eigensolver of the library (host code) — for tests."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    m = A.shape[0]
    ev = np.zeros(m)
    V = np.zeros((m, m))
    _check(_lib.sfairsc_host_symeig(m, A.ctypes.data, ev.ctypes.data, V.ctypes.data))
    return ev, V


def host_symeig_sel(A: np.ndarray, nvec: int):
    """The thick restart's selected-vector variant: all eigenvalues, the nvec smallest eigenvectors."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    m = A.shape[0]
    ev = np.zeros(m)
    V = np.zeros((m, m))
    _check(_lib.sfairsc_host_symeig_sel(m, A.ctypes.data, ev.ctypes.data, V.ctypes.data, int(nvec)))
    return ev, V[:, :nvec]


# --- multi-GPU (row-partitioned) ---------------------------------------

class Comm:
    """An NCCL communicator of the row-partitioned solver (sfairsc_comm)."""

    def __init__(self, uid: bytes, rank: int, nranks: int, device: int):
        if len(uid) != 128:
            raise ValueError("unique id must be 128 bytes")
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        _check(_lib.sfairsc_comm_init(C.cast(buf, C.c_void_p), rank, nranks, device, C.byref(h)))
        self.handle = h
        self.rank, self.nranks, self.device = rank, nranks, device

    def close(self):
        if self.handle:
            _lib.sfairsc_comm_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def comm_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(_lib.sfairsc_comm_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


def comm_from_torch(device: int, group=None) -> Comm:
    """Bootstrap over an initialised torch.distributed process group: rank 0
    creates the NCCL unique id, every rank receives it by broadcast and joins."""
    import torch.distributed as dist
    rank, ws = dist.get_rank(group), dist.get_world_size(group)
    uid = broadcast_uid(comm_unique_id() if rank == 0 else None, group)
    return Comm(uid, rank, ws, device)


def broadcast_uid(uid: bytes | None, group=None) -> bytes:
    """Rank 0's 128-byte NCCL unique id, delivered to every rank of `group`."""
    import torch.distributed as dist
    obj = [uid if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    if not isinstance(obj[0], (bytes, bytearray)) or len(obj[0]) != 128:
        raise RuntimeError("bad unique id broadcast")
    return bytes(obj[0])


def partition_rows(row_ptr: np.ndarray, nparts: int) -> np.ndarray:
    """Contiguous row blocks balanced by nnz + 4 per row (the library's own
    rule for virtual parts): cuts[q] <= rows of part q < cuts[q+1]."""
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    n = len(row_ptr) - 1
    w = row_ptr + 4 * np.arange(n + 1, dtype=np.int64)
    tot = int(w[-1])
    cuts = np.zeros(nparts + 1, dtype=np.int64)
    cuts[-1] = n
    for q in range(1, nparts):
        cuts[q] = max(cuts[q - 1], int(np.searchsorted(w, tot * q // nparts, side="left")))
    return cuts


def row_block(row_ptr, col_idx, values, groups, r0: int, r1: int):
    """The CSR rows [r0, r1) of W (global column indices kept) and their groups."""
    a, b = int(row_ptr[r0]), int(row_ptr[r1])
    rp = (np.asarray(row_ptr[r0:r1 + 1], dtype=np.int64) - a).astype(np.int32)
    return rp, np.ascontiguousarray(col_idx[a:b]), np.ascontiguousarray(values[a:b]), \
        np.ascontiguousarray(np.asarray(groups[r0:r1], dtype=np.int32))
