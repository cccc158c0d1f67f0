"""TEST INFRASTRUCTURE — ctypes access to the CPU checkers. NOT product code.

  liboracle.so         plain-C restatement of the reference algorithm (oracle/oracle.c)
  _ref/libfea_ref.so   the unmodified reference library + extern "C" driver (oracle/ref_driver.cpp)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this package, and only as the checker / CPU baseline. The product
(paper_2012_00585_b200) never imports it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, c_double, c_int, c_int32, c_int64, c_uint64, c_void_p
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libfea_ref.so"
REF_SRC = Path(os.environ.get("FEA_REF_SRC", "/root/reference/proj"))


def build(ref: bool = True) -> None:
    """make the oracle (always) and the reference library (when its sources exist)."""
    subprocess.run(["make", "-s", "-C", str(HERE), "oracle"], check=True)
    if ref and (REF_SRC / "src").is_dir():
        subprocess.run(["make", "-s", "-C", str(HERE), "-j8", "ref", f"REF={REF_SRC}"], check=True)


def _p(a):
    return c_void_p(0) if a is None else c_void_p(a.ctypes.data)


_orc = None
_ref = None


def orc():
    global _orc
    if _orc is None:
        if not ORACLE_SO.exists():
            build(ref=False)
        L = ctypes.CDLL(str(ORACLE_SO))
        L.orc_kval.restype = c_double
        L.orc_kval.argtypes = [c_uint64, c_int64, c_int32, c_int32]
        L.orc_splitmix64.restype = c_uint64
        L.orc_splitmix64.argtypes = [c_uint64]
        L.orc_fill_k.argtypes = [c_uint64, c_int64, c_int32, c_void_p]
        L.orc_fill_k_range.argtypes = [c_uint64, c_int64, c_int64, c_int32, c_void_p]
        L.orc_build_pattern.restype = c_void_p
        L.orc_build_pattern.argtypes = [c_void_p, c_int64, c_int, c_int64, c_int]
        L.orc_pattern_from_arrays.restype = c_void_p
        L.orc_pattern_from_arrays.argtypes = [c_int64, c_void_p, c_void_p]
        L.orc_pattern_free.argtypes = [c_void_p]
        L.orc_pattern_sizes.argtypes = [c_void_p, POINTER(c_int64), POINTER(c_int64), POINTER(c_int64)]
        L.orc_pattern_copy.argtypes = [c_void_p, c_void_p, c_void_p]
        L.orc_count_runs.restype = c_int64
        L.orc_count_runs.argtypes = [c_void_p]
        L.orc_crac_arrays.argtypes = [c_void_p, c_void_p, c_void_p]
        L.orc_locate_csr.restype = c_int64
        L.orc_locate_csr.argtypes = [c_void_p, c_int64, c_int64]
        L.orc_locate_crac.restype = c_int64
        L.orc_locate_crac.argtypes = [c_void_p, c_void_p, c_int64, c_int64]
        L.orc_encode_runs.restype = c_int64
        L.orc_encode_runs.argtypes = [c_void_p, c_int64, c_void_p]
        L.orc_greedy_colouring.restype = c_int
        L.orc_greedy_colouring.argtypes = [c_void_p, c_int64, c_int, c_int64, c_void_p]
        L.orc_assemble_sequential.restype = c_int
        L.orc_assemble_sequential.argtypes = [c_void_p, c_void_p, c_int64, c_int, c_void_p, c_void_p, c_void_p]
        L.orc_assemble_coloured.restype = c_int
        L.orc_assemble_coloured.argtypes = [c_void_p, c_void_p, c_int64, c_int, c_void_p, c_void_p,
                                            c_void_p, c_void_p]
        L.orc_adjacency_new.restype = c_void_p
        L.orc_adjacency_new.argtypes = [c_void_p, c_int64, c_int, c_int64]
        L.orc_adjacency_free.argtypes = [c_void_p]
        L.orc_node_counts.argtypes = [c_void_p, c_int64, c_int64, c_void_p, c_void_p]
        L.orc_node_rows.restype = c_int
        L.orc_node_rows.argtypes = [c_void_p, c_int, c_uint64, c_void_p, c_void_p, c_int64, c_int, c_void_p,
                                    c_void_p, c_void_p]
        _orc = L
    return _orc


class MissingEntry(RuntimeError):
    pass


class Pattern:
    """Oracle SparsityPattern (owns a C orc_pattern)."""

    def __init__(self, handle):
        self._h = c_void_p(handle)
        r, z, u = c_int64(), c_int64(), c_int64()
        orc().orc_pattern_sizes(self._h, ctypes.byref(r), ctypes.byref(z), ctypes.byref(u))
        self.n_rows, self.nnz, self.n_runs = r.value, z.value, u.value

    @classmethod
    def build(cls, conn: np.ndarray, n_nodes: int, d: int) -> "Pattern":
        c = np.ascontiguousarray(conn, dtype=np.int64)
        return cls(orc().orc_build_pattern(_p(c), c.shape[0], c.shape[1], n_nodes, d))

    @classmethod
    def from_arrays(cls, row_ptr, cols) -> "Pattern":
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        cs = np.ascontiguousarray(cols, dtype=np.int64)
        return cls(orc().orc_pattern_from_arrays(len(rp) - 1, _p(rp), _p(cs if len(cs) else np.zeros(1, np.int64))))

    def arrays(self):
        rp = np.empty(self.n_rows + 1, np.int64)
        cs = np.empty(max(self.nnz, 1), np.int64)
        orc().orc_pattern_copy(self._h, _p(rp), _p(cs))
        return rp, cs[: self.nnz]

    def crac(self):
        rp = np.empty(self.n_rows + 1, np.int64)
        ca = np.empty(2 * self.n_runs + 2, np.int64)
        orc().orc_crac_arrays(self._h, _p(rp), _p(ca))
        return rp, ca

    def locate(self, r: int, c: int) -> int:
        return int(orc().orc_locate_csr(self._h, r, c))

    def assemble_sequential(self, elem_dofs, K, values=None):
        ed = np.ascontiguousarray(elem_dofs, dtype=np.int64)
        Kc = np.ascontiguousarray(K, dtype=np.float64)
        v = np.zeros(self.nnz, np.float64) if values is None else values
        err = np.zeros(3, np.int64)
        rc = orc().orc_assemble_sequential(self._h, _p(ed), ed.shape[0], ed.shape[1], _p(Kc),
                                           _p(v), _p(err))
        if rc:
            raise MissingEntry(tuple(int(x) for x in err))
        return v

    def assemble_coloured(self, elem_dofs, K, colour_of, values=None):
        ed = np.ascontiguousarray(elem_dofs, dtype=np.int64)
        Kc = np.ascontiguousarray(K, dtype=np.float64)
        col = np.ascontiguousarray(colour_of, dtype=np.int32)
        v = np.zeros(self.nnz, np.float64) if values is None else values
        err = np.zeros(3, np.int64)
        rc = orc().orc_assemble_coloured(self._h, _p(ed), ed.shape[0], ed.shape[1], _p(Kc),
                                         _p(col), _p(v), _p(err))
        if rc:
            raise MissingEntry(tuple(int(x) for x in err))
        return v

    def __del__(self):
        try:
            if self._h:
                orc().orc_pattern_free(self._h)
        except Exception:
            pass


class Adjacency:
    """Restricted oracle for meshes too large for the full one (SURVEY.md §8c "oracle limits",
    config 5): the reference's node -> element index (pattern.cpp:32-48), node row lengths
    (so the whole int64 row_ptr is checked) and the assembled values of selected node rows
    with the seeded supplier (orc_node_rows: assemble_sequential / colour-vec order)."""

    def __init__(self, conn: np.ndarray, n_nodes: int):
        self._conn = np.ascontiguousarray(conn, dtype=np.int64)  # borrowed by the C side
        self.n_nodes = n_nodes
        self.npe = self._conn.shape[1]
        self._h = c_void_p(orc().orc_adjacency_new(_p(self._conn), self._conn.shape[0], self.npe, n_nodes))

    def node_counts(self, threads: int = 0):
        """(count, runs) per node: node-level row length and CRAC runs."""
        out = np.empty(self.n_nodes, np.int64)
        runs = np.empty(self.n_nodes, np.int64)
        threads = threads or (os.cpu_count() or 1)
        step = max(1 << 14, (self.n_nodes + threads - 1) // threads)
        L = orc()
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda v0: L.orc_node_counts(self._h, v0, min(v0 + step, self.n_nodes),
                                                     c_void_p(out[v0:].ctypes.data), c_void_p(runs[v0:].ctypes.data)),
                        range(0, self.n_nodes, step)))
        return out, runs

    def row_ptrs(self, d: int, threads: int = 0):
        """Whole-matrix (CSR row_ptr, CRAC row_ptr) int64: row (v,k) has d*count(v) entries and
        2*runs(v) col_align entries (build_crac_arrays, formats.cpp:21-41)."""
        c, r = self.node_counts(threads)
        rp = np.zeros(self.n_nodes * d + 1, np.int64)
        rp[1:] = np.cumsum(np.repeat(c * d, d))
        cp = np.zeros(self.n_nodes * d + 1, np.int64)
        cp[1:] = np.cumsum(np.repeat(2 * r, d))
        return rp, cp

    def node_rows(self, nodes, d: int, seed: int, colour_of=None, max_cols: int = 128):
        """(cnt[n], cols[n, max_cols] node ids, vals[n, d, max_cols*d]) of the selected nodes."""
        nd = np.ascontiguousarray(nodes, dtype=np.int64)
        cnt = np.zeros(len(nd), np.int64)
        cols = np.zeros((len(nd), max_cols), np.int64)
        vals = np.zeros((len(nd), d, max_cols * d), np.float64)
        col = None if colour_of is None else np.ascontiguousarray(colour_of, dtype=np.int32)
        if orc().orc_node_rows(self._h, d, seed, _p(col), _p(nd), len(nd), max_cols, _p(cnt), _p(cols), _p(vals)):
            raise ValueError("node row longer than max_cols")
        return cnt, cols, vals

    def __del__(self):
        try:
            if self._h:
                orc().orc_adjacency_free(self._h)
        except Exception:
            pass


def locate_crac(crac_ptr, col_align, r: int, c: int) -> int:
    return int(orc().orc_locate_crac(_p(crac_ptr), _p(col_align), r, c))


def encode_runs(flat):
    f = np.ascontiguousarray(flat, dtype=np.int64)
    out = np.empty(2 * max(len(f), 1), np.int64)
    n = orc().orc_encode_runs(_p(f), len(f), _p(out))
    return [(int(out[2 * i]), int(out[2 * i + 1])) for i in range(n)]


def greedy_colouring(conn, n_nodes: int):
    c = np.ascontiguousarray(conn, dtype=np.int64)
    col = np.empty(c.shape[0], np.int32)
    n = orc().orc_greedy_colouring(_p(c), c.shape[0], c.shape[1], n_nodes, _p(col))
    return col, n


def fill_k(seed: int, n: int, m: int, e0: int = 0, threads: int = 0) -> np.ndarray:
    """Seeded K of elements e0 .. e0+n-1 (orc_kval), filled by `threads` host threads
    (0: all cores; ctypes releases the GIL)."""
    K = np.empty((n, m, m), np.float64)
    if n == 0:
        return K
    threads = threads or (os.cpu_count() or 1)
    step = max(4096, (n + threads - 1) // threads)
    L = orc()
    if threads == 1 or n <= step:
        L.orc_fill_k_range(seed, e0, n, m, _p(K))
        return K
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(lambda a: L.orc_fill_k_range(seed, e0 + a, min(step, n - a), m, c_void_p(K[a:].ctypes.data)),
                    range(0, n, step)))
    return K


# ----------------------------------------------------------------------------
# The unmodified reference library (oracle/_ref/libfea_ref.so)
# ----------------------------------------------------------------------------

METHODS = {"seq": 0, "atomic": 1, "spin": 2, "spin-vec": 3, "colour-vec": 4}
FORMATS = {"csr": 0, "crac": 1}


def ref_available() -> bool:
    if REF_SO.exists():
        return True
    if (REF_SRC / "src").is_dir():
        build(ref=True)
    return REF_SO.exists()


def ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise FileNotFoundError(f"{REF_SO} not built and reference sources absent")
        L = ctypes.CDLL(str(REF_SO))
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_hardware_threads.restype = c_int
        L.ref_problem_new.restype = c_void_p
        L.ref_problem_new.argtypes = [c_void_p, c_int64, c_int, c_int64, c_int, c_int]
        L.ref_problem_from_pattern.restype = c_void_p
        L.ref_problem_from_pattern.argtypes = [c_void_p, c_int64, c_int, c_int64, c_void_p, c_void_p]
        L.ref_problem_free.argtypes = [c_void_p]
        L.ref_pattern_sizes.argtypes = [c_void_p, POINTER(c_int64), POINTER(c_int64), POINTER(c_int64)]
        L.ref_pattern_copy.argtypes = [c_void_p, c_void_p, c_void_p]
        L.ref_crac_copy.argtypes = [c_void_p, c_void_p, c_void_p]
        L.ref_greedy_colouring.restype = c_int
        L.ref_greedy_colouring.argtypes = [c_void_p, c_void_p]
        L.ref_locate.restype = c_int64
        L.ref_locate.argtypes = [c_void_p, c_int, c_int64, c_int64]
        L.ref_assemble.restype = c_int
        L.ref_assemble.argtypes = [c_void_p, c_void_p, c_int, c_int, c_int, c_void_p, c_void_p,
                                   c_int, c_void_p]
        _ref = L
    return _ref


class RefProblem:
    """A problem driven through the reference API (SURVEY.md §8c padded-DofMap recipe)."""

    def __init__(self, conn=None, n_nodes=0, d=1, build_pattern=True, *, handle=None, m=None):
        L = ref()
        if handle is not None:
            self._h = c_void_p(handle)
            self.m = m
        else:
            c = np.ascontiguousarray(conn, dtype=np.int64)
            self._conn = c
            self._h = c_void_p(L.ref_problem_new(_p(c), c.shape[0], c.shape[1], n_nodes, d,
                                                 1 if build_pattern else 0))
            self.m = c.shape[1] * d
        if not self._h:
            raise RuntimeError(L.ref_last_error().decode())
        if build_pattern or handle is not None:
            r, z, u = c_int64(), c_int64(), c_int64()
            L.ref_pattern_sizes(self._h, ctypes.byref(r), ctypes.byref(z), ctypes.byref(u))
            self.n_rows, self.nnz, self.n_runs = r.value, z.value, u.value

    @classmethod
    def from_pattern(cls, elem_dofs, n_rows, row_ptr, cols):
        ed = np.ascontiguousarray(elem_dofs, dtype=np.int64)
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        cs = np.ascontiguousarray(cols, dtype=np.int64)
        h = ref().ref_problem_from_pattern(_p(ed), ed.shape[0], ed.shape[1], n_rows, _p(rp),
                                           _p(cs if len(cs) else np.zeros(1, np.int64)))
        return cls(handle=h, m=ed.shape[1])

    def pattern(self):
        rp = np.empty(self.n_rows + 1, np.int64)
        cs = np.empty(max(self.nnz, 1), np.int64)
        ref().ref_pattern_copy(self._h, _p(rp), _p(cs))
        return rp, cs[: self.nnz]

    def crac(self):
        rp = np.empty(self.n_rows + 1, np.int64)
        ca = np.empty(2 * self.n_runs + 2, np.int64)
        ref().ref_crac_copy(self._h, _p(rp), _p(ca))
        return rp, ca

    def greedy_colouring(self, n_elements: int):
        col = np.empty(n_elements, np.int32)
        n = ref().ref_greedy_colouring(self._h, _p(col))
        return col, n

    def locate(self, fmt: str, r: int, c: int) -> int:
        return int(ref().ref_locate(self._h, FORMATS[fmt], r, c))

    def assemble(self, K, method="seq", fmt="csr", threads=1, colour_of=None, values=None):
        Kc = np.ascontiguousarray(K, dtype=np.float64)
        v = np.zeros(self.nnz, np.float64) if values is None else values
        col = None if colour_of is None else np.ascontiguousarray(colour_of, dtype=np.int32)
        rc = ref().ref_assemble(self._h, _p(Kc), METHODS[method], FORMATS[fmt], threads, _p(col),
                                _p(v), 0, c_void_p(0))
        if rc:
            raise MissingEntry(ref().ref_last_error().decode())
        return v

    def time(self, K, method="seq", fmt="csr", threads=1, colour_of=None, runs=5):
        """fea::time_assembly (bench.hpp:98-113): untimed reset + warm-up, then `runs` timed µs."""
        Kc = np.ascontiguousarray(K, dtype=np.float64)
        col = None if colour_of is None else np.ascontiguousarray(colour_of, dtype=np.int32)
        t = np.zeros(runs, np.float64)
        rc = ref().ref_assemble(self._h, _p(Kc), METHODS[method], FORMATS[fmt], threads, _p(col),
                                c_void_p(0), runs, _p(t))
        if rc:
            raise RuntimeError(ref().ref_last_error().decode())
        return t

    def __del__(self):
        try:
            if self._h:
                ref().ref_problem_free(self._h)
        except Exception:
            pass


def hardware_threads() -> int:
    return int(ref().ref_hardware_threads())


def ref_structured_element_nodes(n: int, p: int, d: int = 1):
    """(element_nodes (E, (p+1)^2), n_nodes) from the reference's build_dof_map(generate_structured(n), p, d)."""
    L = ref()
    L.ref_structured_element_nodes.restype = c_int
    L.ref_structured_element_nodes.argtypes = [c_int64, c_int, c_int, c_void_p, POINTER(c_int64),
                                               POINTER(c_int64), POINTER(c_int64)]
    E, npe, nn = c_int64(), c_int64(), c_int64()
    if L.ref_structured_element_nodes(n, p, d, c_void_p(0), ctypes.byref(E), ctypes.byref(npe), ctypes.byref(nn)):
        raise RuntimeError(L.ref_last_error().decode())
    out = np.empty((E.value, npe.value), np.int64)
    L.ref_structured_element_nodes(n, p, d, _p(out), ctypes.byref(E), ctypes.byref(npe), ctypes.byref(nn))
    return out, nn.value


def ref_speed_factor(t_seq: float, t_method: float) -> float:
    L = ref()
    L.ref_speed_factor.restype = c_double
    L.ref_speed_factor.argtypes = [c_double, c_double]
    return float(L.ref_speed_factor(t_seq, t_method))
