"""paper_1709_08625_b200 — thin Python binding of libhcov.so (include/hcov.h).

Argument marshalling only: every step of the likelihood path runs in the CUDA kernels of
``csrc/``.  PyTorch supplies device memory and the current stream.  There is no CPU fallback:
``lib()`` raises if the shared library is missing and every compute entry point requires CUDA
tensors.  Names follow the C ABI (hcov_build_tree, hcov_assemble, hcov_cholesky, hcov_loglik,
hcov_eval, hcov_mle_batch, hcov_sample, hcov_columns).
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HCOV_LIB") or os.path.join(_HERE, "libhcov.so")   # HCOV_LIB: an in-tree build variant (experiments)

HCOV_OK = 0
STATUS = {0: "ok", 1: "invalid argument", 2: "empty input", 3: "not SPD", 4: "out of memory",
          5: "CUDA error", 6: "rank capacity exceeded", 7: "invalid call order"}
ND_H, ND_R, ND_T = 0, 1, 2


class HcovError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"{where}: {STATUS.get(code, code)} ({code})")
        self.code = code


class Theta(ctypes.Structure):
    _fields_ = [("sigma2", ctypes.c_double), ("ell", ctypes.c_double), ("nu", ctypes.c_double),
                ("nugget", ctypes.c_double)]


class Trunc(ctypes.Structure):
    _fields_ = [("eps", ctypes.c_double), ("kmax", ctypes.c_int32), ("kcap", ctypes.c_int32)]


class Result(ctypes.Structure):
    _fields_ = [("loglik", ctypes.c_double), ("logdet", ctypes.c_double), ("quad", ctypes.c_double),
                ("n", ctypes.c_int64), ("max_rank", ctypes.c_int32), ("cap_binds", ctypes.c_int32),
                ("min_pivot", ctypes.c_double), ("fail_leaf", ctypes.c_int64), ("acc_loss", ctypes.c_int32),
                ("interm_cuts", ctypes.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class TreeInfo(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("n_pad", ctypes.c_int64), ("depth", ctypes.c_int32),
                ("leaf_size", ctypes.c_int32), ("n_leaves", ctypes.c_int64), ("n_dense_tiles", ctypes.c_int64),
                ("n_lowrank", ctypes.c_int64), ("n_tasks", ctypes.c_int64), ("n_waves", ctypes.c_int64),
                ("eta", ctypes.c_double), ("uv_elems", ctypes.c_int64), ("w_elems", ctypes.c_int64),
                ("slot_a", ctypes.c_int64), ("slot_b", ctypes.c_int64), ("n_cores", ctypes.c_int64),
                ("n_edges", ctypes.c_int64), ("n_xterm", ctypes.c_int64), ("max_mq", ctypes.c_int64),
                ("tree_on_device", ctypes.c_int32), ("geo_ms", ctypes.c_double), ("dim", ctypes.c_int32)]


class TreeOpts(ctypes.Structure):
    _fields_ = [("leaf_size", ctypes.c_int32), ("eta", ctypes.c_double), ("dense_below", ctypes.c_int32),
                ("factor_trunc", ctypes.c_int32), ("dim", ctypes.c_int32)]


class Prof(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_int64), ("n_classes", ctypes.c_int32), ("n_task_types", ctypes.c_int32),
                ("count", ctypes.c_int64 * 16), ("ms", ctypes.c_double * 16),
                ("task_busy_ms", ctypes.c_double * 16), ("task_count", ctypes.c_double * 16),
                ("flop", ctypes.c_double * 8), ("phase_ms", ctypes.c_double * 16),
                ("phase_cls_ms", ctypes.c_double * 64)]


# name -> (restype, argtypes) ; every symbol declared in include/hcov.h
_P, _I32, _I64, _D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
_SIGS = {
    "hcov_build_tree": (_I32, [_P, _I64, _I32, _D, _I32, _P, _P]),
    "hcov_build_tree_host": (_I32, [_P, _I64, _I32, _D, _I32, _P]),
    "hcov_build_tree_ex": (_I32, [_P, _I64, _P, _P, _P]),
    "hcov_build_tree_host_ex": (_I32, [_P, _I64, _P, _P]),
    "hcov_tree_get_info": (_I32, [_P, _P]),
    "hcov_tree_blocks": (_I32, [_P, _P, _I64, _P]),
    "hcov_tree_bbox": (_I32, [_P, _P, _I64]),
    "hcov_tree_tasks": (_I32, [_P, _P, _I64, _P]),
    "hcov_tree_succ": (_I32, [_P, _P, _P, _I64, _P]),
    "hcov_tree_perm": (_I32, [_P, _P]),
    "hcov_assemble": (_I32, [_P, _P, _P, _P, _P]),
    "hcov_cholesky": (_I32, [_P, _P, _P]),
    "hcov_loglik": (_I32, [_P, _P, _P, _P]),
    "hcov_eval": (_I32, [_P, _P, _P, _P, _P, _P]),
    "hcov_mle_batch": (_I32, [_P, _P, _P, _I32, _P, _P, _P, _P]),
    "hcov_sample": (_I32, [_P, _P, _P, _P]),
    "hcov_columns": (_I32, [_P, _P, _I32, _P, _P]),
    "hcov_hmat_storage": (_I32, [_P, _P, _P, _P]),
    "hcov_hmat_mem_info": (_I32, [_P, _P]),
    "hcov_cov_columns": (_I32, [_P, _P, _P, _I32, _P, _P]),
    "hcov_forward_solve": (_I32, [_P, _P, _P, _P]),
    "hcov_backsolve": (_I32, [_P, _P, _P, _P]),
    "hcov_solve": (_I32, [_P, _P, _P, _P]),
    "hcov_ldl_diag": (_I32, [_P, _P, _P]),
    "hcov_matvec": (_I32, [_P, _P, _P, _P]),
    "hcov_pcg": (_I32, [_P, _P, _P, _P, _I32, _D, _P, _P, _P]),
    "hcov_norm2_diff": (_I32, [_P, _P, _I32, ctypes.c_uint64, _P, _P]),
    "hcov_inv_error": (_I32, [_P, _P, _I32, ctypes.c_uint64, _P, _P]),
    "hcov_trace_inv": (_I32, [_P, _P, _P, _P]),
    "hcov_model_flops": (_I32, [_P, _P]),
    "hcov_tree_last_eval": (_I32, [_P, _P]),
    "hcov_prof_control": (_I32, [_I32, _I32]),
    "hcov_prof_read": (_I32, [_P]),
    "hcov_prof_class_name": (ctypes.c_char_p, [_I32]),
    "hcov_prof_task_name": (ctypes.c_char_p, [_I32]),
    "hcov_test_truncate": (_I32, [_P, _P, _I64, _I32, _D, _I32, _I32, _I32, _P, _P, _P]),
    "hcov_tree_free": (None, [_P]),
    "hcov_hmat_free": (None, [_P]),
    "hcov_status_string": (ctypes.c_char_p, [_I32]),
}
_lib = None


def lib() -> ctypes.CDLL:
    """Load libhcov.so (built in-tree by build.py / __graft_entry__.build()). Fails loudly."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libhcov.so not built ({LIB_PATH}); run `python -m paper_1709_08625_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(code: int, where: str):
    if code != HCOV_OK:
        raise HcovError(code, where)


def _stream(stream=None):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _dev_f64(x, n=None, name="array"):
    import torch
    if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float64 and x.is_contiguous()):
        raise TypeError(f"{name} must be a contiguous float64 CUDA tensor")
    if n is not None and x.numel() != n:
        raise ValueError(f"{name}: expected {n} elements, got {x.numel()}")
    return ctypes.c_void_p(x.data_ptr())


class Tree:
    """Cluster tree + block tree + theta-independent schedule (hcov_tree)."""

    def __init__(self, s, eta: float = 2.0, dense_below: int = 32, leaf_size: int = 32, stream=None,
                 factor_trunc: bool = False):
        """factor_trunc: the SPD-preserving H-Cholesky variant (hcov_tree_opts.factor_trunc, R27)."""
        L = lib()
        h = ctypes.c_void_p()
        if len(s.shape) != 2 or s.shape[1] not in (2, 3):
            raise ValueError("locations must be n x 2, or n x 3 (the 3-D variant)")
        self.dim = int(s.shape[1])
        o = TreeOpts(leaf_size, eta, dense_below, 1 if factor_trunc else 0, self.dim)
        self.factor_trunc = bool(factor_trunc)
        if isinstance(s, np.ndarray):
            a = np.ascontiguousarray(s, dtype=np.float64)
            self.n = a.shape[0]
            _check(L.hcov_build_tree_host_ex(a.ctypes.data, self.n, ctypes.byref(o), ctypes.byref(h)),
                   "hcov_build_tree_host_ex")
        else:
            self.n = s.shape[0]
            _check(L.hcov_build_tree_ex(_dev_f64(s, self.dim * self.n, "s"), self.n, ctypes.byref(o), _stream(stream),
                                        ctypes.byref(h)), "hcov_build_tree_ex")
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.hcov_tree_free(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def info(self) -> dict:
        i = TreeInfo()
        _check(lib().hcov_tree_get_info(self._h, ctypes.byref(i)), "hcov_tree_get_info")
        return {k: getattr(i, k) for k, _ in i._fields_}

    def perm_i2e(self) -> np.ndarray:
        npad = self.info()["n_pad"]
        p = np.empty(npad, dtype=np.int64)
        _check(lib().hcov_tree_perm(self._h, p.ctypes.data), "hcov_tree_perm")
        return p

    def blocks(self) -> np.ndarray:
        cnt = ctypes.c_int64()
        _check(lib().hcov_tree_blocks(self._h, None, 0, ctypes.byref(cnt)), "hcov_tree_blocks")
        out = np.empty((cnt.value, 4), dtype=np.int32)
        _check(lib().hcov_tree_blocks(self._h, out.ctypes.data, cnt.value, ctypes.byref(cnt)), "hcov_tree_blocks")
        return out

    def tasks(self) -> np.ndarray:
        """hcov_tree_tasks: (n_tasks, 6) int32 = type, phase, a, b, c, d."""
        cnt = ctypes.c_int64()
        _check(lib().hcov_tree_tasks(self._h, None, 0, ctypes.byref(cnt)), "hcov_tree_tasks")
        out = np.empty((cnt.value, 6), dtype=np.int32)
        _check(lib().hcov_tree_tasks(self._h, out.ctypes.data, cnt.value, ctypes.byref(cnt)), "hcov_tree_tasks")
        return out

    def succ(self):
        """hcov_tree_succ: (off[n_tasks + 1], succ[]) CSR of the task DAG."""
        cnt = ctypes.c_int64()
        _check(lib().hcov_tree_succ(self._h, None, None, 0, ctypes.byref(cnt)), "hcov_tree_succ")
        off = np.empty(self.info()["n_tasks"] + 1, dtype=np.int32)
        sc = np.empty(max(1, cnt.value), dtype=np.int32)
        _check(lib().hcov_tree_succ(self._h, off.ctypes.data, sc.ctypes.data, sc.size, ctypes.byref(cnt)),
               "hcov_tree_succ")
        return off, sc[:cnt.value]

    def bbox(self) -> np.ndarray:
        d = self.info()["depth"]
        nc = (2 << d) - 1
        out = np.empty((nc, 2 * self.dim), dtype=np.float64)
        _check(lib().hcov_tree_bbox(self._h, out.ctypes.data, out.size), "hcov_tree_bbox")
        return out


class _Borrowed:
    """A borrowed hcov_hmat (not freed by Python)."""

    def __init__(self, tree, h):
        self.tree, self._h = tree, h

    model_flops = None
    storage = None
    mem_info = None


def last_eval(tree: "Tree"):
    """hcov_tree_last_eval: the factored H-matrix of the last eval_loglik on this tree (borrowed)."""
    h = ctypes.c_void_p()
    _check(lib().hcov_tree_last_eval(tree.handle, ctypes.byref(h)), "hcov_tree_last_eval")
    b = _Borrowed(tree, h)
    b.model_flops = HMatrix.model_flops.__get__(b)
    b.storage = HMatrix.storage.__get__(b)
    b.mem_info = HMatrix.mem_info.__get__(b)
    return b


def build_tree(s, eta: float = 2.0, dense_below: int = 32, stream=None) -> Tree:
    return Tree(s, eta=eta, dense_below=dense_below, stream=stream)


class HMatrix:
    """Device H-matrix (hcov_hmat): C~ after assemble, L~ after cholesky."""

    def __init__(self, tree: Tree, theta, eps: float, kmax: int = 0, kcap: int = 0, stream=None):
        self.tree = tree
        h = ctypes.c_void_p()
        th = Theta(*theta)
        tr = Trunc(eps, kmax, kcap)
        _check(lib().hcov_assemble(tree.handle, ctypes.byref(th), ctypes.byref(tr), _stream(stream), ctypes.byref(h)),
               "hcov_assemble")
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.hcov_hmat_free(self._h)
            self._h = None

    def cholesky(self, stream=None) -> int:
        fl = ctypes.c_int64(-1)
        code = lib().hcov_cholesky(self._h, _stream(stream), ctypes.byref(fl))
        _check(code, "hcov_cholesky")
        return fl.value

    def loglik(self, Z, stream=None) -> dict:
        r = Result()
        _check(lib().hcov_loglik(self._h, _dev_f64(Z, self.tree.n, "Z"), _stream(stream), ctypes.byref(r)),
               "hcov_loglik")
        return r.as_dict()

    def sample(self, xi, stream=None):
        import torch
        Z = torch.empty_like(xi)
        _check(lib().hcov_sample(self._h, _dev_f64(xi, self.tree.n, "xi"), _dev_f64(Z), _stream(stream)),
               "hcov_sample")
        return Z

    def columns(self, cols: Sequence[int], stream=None):
        import torch
        c = np.ascontiguousarray(cols, dtype=np.int64)
        out = torch.empty((len(c), self.tree.n), dtype=torch.float64, device="cuda")
        _check(lib().hcov_columns(self._h, c.ctypes.data, len(c), _dev_f64(out), _stream(stream)), "hcov_columns")
        return out.T   # n x m, external rows

    def _vec_op(self, fn, x, name, stream=None):
        import torch
        y = torch.empty_like(x)
        _check(getattr(lib(), fn)(self._h, _dev_f64(x, self.tree.n, "x"), _dev_f64(y), _stream(stream)), fn)
        return y

    def forward_solve(self, z, stream=None):
        """hcov_forward_solve: v = P L~^{-1} P^T z (external order)."""
        return self._vec_op("hcov_forward_solve", z, "z", stream)

    def ldl_diag(self, stream=None):
        """hcov_ldl_diag: D of the point-wise LDL^T form (n, external order) of the factored matrix."""
        import torch
        D = torch.empty(self.tree.n, dtype=torch.float64, device="cuda")
        _check(lib().hcov_ldl_diag(self._h, _dev_f64(D), _stream(stream)), "hcov_ldl_diag")
        return D

    def backsolve(self, v, stream=None):
        """hcov_backsolve: u = P L~^{-T} P^T v (external order)."""
        return self._vec_op("hcov_backsolve", v, "v", stream)

    def solve(self, b, stream=None):
        """hcov_solve: x = C~^{-1} b through the factor."""
        return self._vec_op("hcov_solve", b, "b", stream)

    def matvec(self, x, stream=None):
        """hcov_matvec: y = C~ x (assembled, not factored)."""
        return self._vec_op("hcov_matvec", x, "x", stream)

    def model_flops(self) -> dict:
        """hcov_model_flops: SURVEY Sec. 8(d) method-work model at the measured ranks (factored)."""
        o = np.zeros(8)
        _check(lib().hcov_model_flops(self._h, o.ctypes.data), "hcov_model_flops")
        return dict(zip(["total", "truncation", "products", "tile", "solves", "potrf", "aca_truncation",
                         "root_solve"], o.tolist()))

    def storage(self) -> dict:
        d, l, m = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
        _check(lib().hcov_hmat_storage(self._h, ctypes.byref(d), ctypes.byref(l), ctypes.byref(m)), "hcov_hmat_storage")
        return {"dense_bytes": d.value, "lowrank_bytes": l.value, "max_rank": m.value}

    def mem_info(self) -> dict:
        """hcov_hmat_mem_info: device bytes of the handle's pools and their use by the last run."""
        o = np.zeros(8, dtype=np.int64)
        _check(lib().hcov_hmat_mem_info(self._h, o.ctypes.data), "hcov_hmat_mem_info")
        return dict(zip(["tiles", "uv", "cores", "w_cap", "p_cap", "w_used", "p_used", "overflows"],
                        [int(x) for x in o]))


def cov_columns(tree: Tree, theta, cols: Sequence[int], stream=None):
    """hcov_cov_columns: exact Eq. (3) columns C e_j on the device (n x m, external rows)."""
    import torch
    c = np.ascontiguousarray(cols, dtype=np.int64)
    out = torch.empty((len(c), tree.n), dtype=torch.float64, device="cuda")
    th = Theta(*theta)
    _check(lib().hcov_cov_columns(tree.handle, ctypes.byref(th), c.ctypes.data, len(c), _dev_f64(out),
                                  _stream(stream)), "hcov_cov_columns")
    return out.T


def eval_loglik(tree: Tree, theta, Z, eps: float, kmax: int = 0, kcap: int = 0, stream=None) -> dict:
    """hcov_eval: assemble + H-Cholesky + log det + forward solve. Raises HcovError(3) if not SPD."""
    r = Result()
    th = Theta(*theta)
    tr = Trunc(eps, kmax, kcap)
    code = lib().hcov_eval(tree.handle, ctypes.byref(th), ctypes.byref(tr), _dev_f64(Z, tree.n, "Z"),
                           _stream(stream), ctypes.byref(r))
    d = r.as_dict()
    d["status"] = code
    if code not in (HCOV_OK, 3, 6):
        raise HcovError(code, "hcov_eval")
    return d


def pcg(A: "HMatrix", M: "HMatrix", b, maxit: int = 150, tol: float = 1e-6, stream=None):
    """hcov_pcg: C~ x = b by CG preconditioned with the H-Cholesky factor M (listing PAPER.md:550-555).
    Returns (x, iterations, relative residual)."""
    import torch
    x = torch.empty_like(b)
    it, rr = ctypes.c_int32(), ctypes.c_double()
    _check(lib().hcov_pcg(A._h, M._h, _dev_f64(b, A.tree.n, "b"), _dev_f64(x), maxit, tol, _stream(stream),
                          ctypes.byref(it), ctypes.byref(rr)), "hcov_pcg")
    return x, it.value, rr.value


def norm2_diff(A: "HMatrix", B: "HMatrix", iters: int = 30, seed: int = 1, stream=None) -> float:
    """hcov_norm2_diff: ||A~ - B~||_2 of two assembled H-matrices on the same points."""
    o = ctypes.c_double()
    _check(lib().hcov_norm2_diff(A._h, B._h, iters, seed, _stream(stream), ctypes.byref(o)), "hcov_norm2_diff")
    return o.value


def inv_error(A: "HMatrix", M: "HMatrix", iters: int = 30, seed: int = 1, stream=None) -> float:
    """hcov_inv_error: ||I - M^{-1} A~||_2 (A assembled, M factored)."""
    o = ctypes.c_double()
    _check(lib().hcov_inv_error(A._h, M._h, iters, seed, _stream(stream), ctypes.byref(o)), "hcov_inv_error")
    return o.value


def trace_inv(M: "HMatrix", A: "HMatrix", stream=None) -> float:
    """hcov_trace_inv: tr(M^{-1} A) (M factored, A assembled)."""
    o = ctypes.c_double()
    _check(lib().hcov_trace_inv(M._h, A._h, _stream(stream), ctypes.byref(o)), "hcov_trace_inv")
    return o.value


def kld(tree: Tree, exact_tree: Tree, theta, eps: float, kmax: int = 0, kcap: int = 0) -> dict:
    """Sec. 4 diagnostics of C~ (eps, kmax) against the exact C: KLD,
    ||C - C~||_2 and ||C C~^{-1} - I||_2.  exact_tree: the same points with eta = 0 (all dense, C~ = C).
    Every quantity is computed by the library's kernels; only the closing arithmetic is here."""
    n = tree.n
    Ce = HMatrix(exact_tree, theta, 0.0)            # assembled exact C
    Cf = HMatrix(exact_tree, theta, 0.0)
    Cf.cholesky()
    import torch
    ld_c = Cf.loglik(torch.zeros(n, dtype=torch.float64, device="cuda"))["logdet"]
    A = HMatrix(tree, theta, eps, kmax, kcap)       # assembled C~
    M = HMatrix(tree, theta, eps, kmax, kcap)
    M.cholesky()
    ld_t = M.loglik(torch.zeros(n, dtype=torch.float64, device="cuda"))["logdet"]
    tr = trace_inv(M, Ce)
    return {"kld": 0.5 * (tr - n + ld_t - ld_c), "trace": tr, "logdet_C": ld_c, "logdet_Ct": ld_t,
            "norm2_C_minus_Ct": norm2_diff(Ce, A), "norm2_C_Ctinv_minus_I": inv_error(Ce, M),
            "max_rank": A.storage()["max_rank"]}


def mle_batch(tree: Tree, Z, thetas, eps: float, kmax: int = 0, kcap: int = 0, stream=None):
    """hcov_mle_batch: returns (loglik[m], status[m]); rejected candidates get -inf."""
    m = len(thetas)
    arr = (Theta * m)(*[Theta(*t) for t in thetas])
    tr = Trunc(eps, kmax, kcap)
    ll = np.empty(m, dtype=np.float64)
    st = np.empty(m, dtype=np.int32)
    _check(lib().hcov_mle_batch(tree.handle, _dev_f64(Z, tree.n, "Z"), ctypes.cast(arr, ctypes.c_void_p), m,
                                ctypes.byref(tr), _stream(stream), ll.ctypes.data, st.ctypes.data), "hcov_mle_batch")
    return ll, st


def prof_control(enable_events: bool = False, reset: bool = True) -> None:
    """hcov_prof_control: launch counting is always on; events time every launch by class."""
    _check(lib().hcov_prof_control(int(enable_events), int(reset)), "hcov_prof_control")


def prof_read() -> dict:
    """hcov_prof_read: launches, per-class device ms, engine busy ms / counts per task type,
    algorithmic flop per flop class."""
    p = Prof()
    _check(lib().hcov_prof_read(ctypes.byref(p)), "hcov_prof_read")
    names = [lib().hcov_prof_class_name(k).decode() for k in range(p.n_classes)]
    tnames = [lib().hcov_prof_task_name(k).decode() for k in range(p.n_task_types)]
    return {"launches": p.launches, "count": {nm: p.count[k] for k, nm in enumerate(names)},
            "ms": {nm: p.ms[k] for k, nm in enumerate(names)},
            "task_busy_ms": {nm: p.task_busy_ms[k] for k, nm in enumerate(tnames)},
            "task_count": {nm: int(p.task_count[k]) for k, nm in enumerate(tnames)},
            "flop": {nm: p.flop[k] for k, nm in enumerate(FLOP_CLASSES)},
            "phase_ms": {nm: p.phase_ms[k] for k, nm in enumerate(PHASES) if nm},
            "phase_cls_ms": {f"{cls}:{nm}": round(p.phase_cls_ms[k + 16 * ci], 1)
                             for ci, cls in enumerate(["m<=64", "m<=256", "m<=1024", "m>1024"])
                             for k, nm in enumerate(PHASES) if nm and p.phase_cls_ms[k + 16 * ci] > 0}}


PHASES = ["panel_qr", "core_product", "pivoted_qr", "svd", "q_apply", "aca_full", "dense_updates", "",
          "aca_partial", "gang_local_qr", "gang_stack_qr", "gang_core", "gang_rows", "gang_wait", "rapp_append", "dense_gemm"]


FLOP_CLASSES = ["assembly_evals", "tile", "truncation", "solve", "products"]


def roofline(prof: dict, peaks: dict) -> dict:
    """Roofline entry of the dominant kernel class (largest device time).  Filled in by the
    per-class algorithmic work model; see bench.py."""
    ms = prof["ms"]
    top = max(ms, key=lambda k: ms[k]) if ms else None
    return {"kernel": top, "ms": ms.get(top), "launches": prof["count"].get(top)}


def test_truncate(X, Y, eps: float, kmax: int = 0, rlim: int = 64, path: int = 1):
    """hcov_test_truncate: truncation A6 of X Y^T on one CTA; returns (U, V, rank, cap_bound, overflow)."""
    import torch
    m, R = X.shape
    Xc = X.T.contiguous()   # column-major
    Yc = Y.T.contiguous()
    U = torch.zeros((rlim, m), dtype=torch.float64, device="cuda")
    V = torch.zeros((rlim, m), dtype=torch.float64, device="cuda")
    out = np.zeros(3, dtype=np.int32)
    _check(lib().hcov_test_truncate(_dev_f64(Xc), _dev_f64(Yc), m, R, eps, kmax, rlim, path, _dev_f64(U), _dev_f64(V),
                                    out.ctypes.data), "hcov_test_truncate")
    r = int(out[0])
    return U[:r].T, V[:r].T, r, int(out[1]), int(out[2])
