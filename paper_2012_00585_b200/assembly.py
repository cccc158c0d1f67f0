"""Python host interface over the C ABI (used by bench.py and the tests).

Mirrors the reference's assembly surface (proj/include/fea/*.hpp):
  * ``Plan``                    — SparsityPattern + CsrMatrix/CracMatrix construction
                                  (build_pattern pattern.cpp:24-108, formats.hpp:157/:268) and the
                                  cached slot map; one plan serves CSR and CRAC (same values order,
                                  verify.cpp:30-31)
  * ``Plan.assemble(K, ...)``   — assemble_atomic / assemble_sequential /
                                  assemble_coloured_vectorized (assembly.hpp:112-195)
  * ``AssemblyError``           — fea::AssemblyError (types.hpp:31-33): missing entry, bad colouring
Device memory and streams come from torch; torch types never cross the C ABI.
"""
from __future__ import annotations

import ctypes
from ctypes import byref, c_int32, c_int64, c_void_p

import numpy as np

from . import _native as N

STRATEGIES = {"atomic": N.FEA_ATOMIC, "sorted": N.FEA_DET_SORTED, "colour": N.FEA_DET_COLOUR,
              "colour_passes": N.FEA_DET_COLOUR}
# "colour": colour-ordered segmented reduction; "colour_passes": one launch per colour
# (element owner, plain adds). Both are bit-identical to assemble_coloured_vectorized.
_EXTRA_FLAGS = {"colour_passes": N.FEA_COLOUR_PASSES}


class FeaError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


class AssemblyError(FeaError):
    """fea::AssemblyError: coefficient missing from the pattern, or invalid colouring."""


def _check(status: int) -> None:
    if status == N.FEA_OK:
        return
    msg = N.last_error()
    if status in (N.FEA_ERR_MISSING_ENTRY, N.FEA_ERR_INVALID_COLOURING):
        raise AssemblyError(status, msg)
    if status == N.FEA_ERR_OOM:
        raise MemoryError(msg)
    if status == N.FEA_ERR_INVALID:
        raise ValueError(msg)
    raise FeaError(status, msg)


def _ptr(x) -> c_void_p:
    """Raw pointer of a numpy array or torch tensor (contiguous)."""
    if x is None:
        return c_void_p(0)
    if isinstance(x, np.ndarray):
        assert x.flags["C_CONTIGUOUS"]
        return c_void_p(x.ctypes.data)
    assert x.is_contiguous()
    return c_void_p(x.data_ptr())


def _stream_ptr(stream, device: int | None = None) -> c_void_p:
    if stream is None:
        import torch
        stream = torch.cuda.current_stream(device)
    return c_void_p(stream.cuda_stream)


def _as_int64_dofs(elem_dofs):
    if isinstance(elem_dofs, np.ndarray):
        a = np.ascontiguousarray(elem_dofs, dtype=np.int64)
        return a, a.shape[0] if a.ndim == 2 else 0, a.shape[1] if a.ndim == 2 else 0
    import torch
    t = elem_dofs.to(torch.int64).contiguous()
    return t, t.shape[0], t.shape[1]


class Plan:
    """Symbolic phase + slot map on one GPU for E elements with m DOFs each.

    elem_dofs : (E, m) int64 — ElementDofs::flat of every element (host numpy or torch tensor)
    n_rows    : global number of rows (DofMap::n_dofs)
    dofs_per_node : d (DOFs v*d..v*d+d-1 per node, dof_map.hpp:59); detected, 1 if absent
    row_range : owned [row_begin, row_end) for row-partitioned assembly (default: all rows)
    k_compact : K holds only the kept elements (ascending id) instead of all E
    """

    def __init__(self, elem_dofs, n_rows: int, dofs_per_node: int = 1, row_range=None,
                 device: int = 0, k_compact: bool = False, _handle=None):
        self._lib = N.lib()
        self.device = device
        self._h = c_void_p(0)
        self.m = None
        self._krows = None
        if _handle is not None:
            self._h = _handle
        else:
            dofs, E, m = _as_int64_dofs(elem_dofs)
            self.m, self._krows = m, (None if k_compact else E)
            rb, re = (0, n_rows) if row_range is None else row_range
            flags = N.FEA_PLAN_K_COMPACT if k_compact else 0
            h = c_void_p(0)
            _check(self._lib.fea_plan_create(device, _ptr(dofs), E, m, n_rows, dofs_per_node, rb, re,
                                             flags, byref(h)))
            self._h = h
        self._refresh()

    @classmethod
    def with_pattern(cls, elem_dofs, n_rows: int, row_ptr, idx, fmt: str = "csr", device: int = 0):
        """Plan against a caller-supplied CSR (row_ptr, cols) or CRAC (row_ptr, col_align) pattern."""
        lib = N.lib()
        dofs, E, m = _as_int64_dofs(elem_dofs)

        def arr(x):  # host arrays like the reference's, or device tensors used in place
            if hasattr(x, "is_cuda"):
                import torch
                assert x.is_cuda and x.dtype == torch.int64 and x.is_contiguous(), \
                    "device pattern arrays must be contiguous cuda int64 tensors"
                return x
            return np.ascontiguousarray(x, dtype=np.int64)

        rp, ix = arr(row_ptr), arr(idx)
        f = N.FEA_FORMAT_CSR if fmt == "csr" else N.FEA_FORMAT_CRAC
        h = c_void_p(0)
        _check(lib.fea_plan_create_with_pattern(device, _ptr(dofs), E, m, n_rows, f, _ptr(rp),
                                                _ptr(ix), byref(h)))
        plan = cls(None, n_rows, device=device, _handle=h)
        plan.m, plan._krows = m, E
        return plan

    def _refresh(self):
        r, z, u, e = c_int64(), c_int64(), c_int64(), c_int64()
        _check(self._lib.fea_plan_sizes(self._h, byref(r), byref(z), byref(u), byref(e)))
        self.n_rows, self.nnz, self.n_runs, self.n_elements = r.value, z.value, u.value, e.value
        d, npe, meta = c_int32(), c_int32(), c_int64()
        _check(self._lib.fea_plan_info(self._h, byref(d), byref(npe), byref(meta)))
        self.dofs_per_node, self.nodes_per_element, self.metadata_bytes = d.value, npe.value, meta.value
        if self._krows is None:  # K holds the kept elements only (FEA_PLAN_K_COMPACT)
            self._krows = self.n_elements

    # argument checks before raw pointers cross the ABI (a short or mistyped buffer would be
    # read / written out of bounds by the kernels)
    def _check_k(self, K, host: bool = False):
        shape = (self._krows, self.m, self.m)
        if host:
            assert isinstance(K, np.ndarray) and K.dtype == np.float64 and K.flags["C_CONTIGUOUS"], \
                "K must be a C-contiguous float64 numpy array"
            assert K.size == self._krows * self.m * self.m, f"K must hold {shape} doubles"
            return
        import torch
        assert K.dtype == torch.float64 and K.is_cuda and K.is_contiguous(), "K must be contiguous cuda float64"
        assert K.device.index == self.device, f"K must be on cuda:{self.device}"
        assert K.numel() == self._krows * self.m * self.m, f"K must hold {shape} doubles"

    def _check_values(self, values, host: bool = False):
        if host:
            assert isinstance(values, np.ndarray) and values.dtype == np.float64 and values.flags["C_CONTIGUOUS"]
            assert values.size >= self.nnz, f"values must hold >= {self.nnz} doubles"
            return
        import torch
        assert values.dtype == torch.float64 and values.is_cuda and values.is_contiguous()
        assert values.device.index == self.device, f"values must be on cuda:{self.device}"
        assert values.numel() >= self.nnz, f"values must hold >= {self.nnz} doubles"

    # -- symbolic outputs -------------------------------------------------
    def csr(self):
        row_ptr = np.empty(self.n_rows + 1, np.int64)
        cols = np.empty(max(self.nnz, 1), np.int64)
        _check(self._lib.fea_plan_copy_csr(self._h, _ptr(row_ptr), _ptr(cols)))
        return row_ptr, cols[: self.nnz]

    def row_ptr(self):
        """CSR row_ptr only (host int64[n_rows+1])."""
        row_ptr = np.empty(self.n_rows + 1, np.int64)
        _check(self._lib.fea_plan_copy_csr(self._h, _ptr(row_ptr), c_void_p(0)))
        return row_ptr

    def csr_device(self):
        """CSR arrays as device tensors (written in place: no host or device temporaries)."""
        import torch
        dev = f"cuda:{self.device}"
        row_ptr = torch.empty(self.n_rows + 1, dtype=torch.int64, device=dev)
        cols = torch.empty(max(self.nnz, 1), dtype=torch.int64, device=dev)
        _check(self._lib.fea_plan_copy_csr(self._h, _ptr(row_ptr), _ptr(cols)))
        return row_ptr, cols[: self.nnz]

    def crac_device(self):
        """CRAC arrays as device tensors."""
        import torch
        dev = f"cuda:{self.device}"
        row_ptr = torch.empty(self.n_rows + 1, dtype=torch.int64, device=dev)
        col_align = torch.empty(2 * self.n_runs + 2, dtype=torch.int64, device=dev)
        _check(self._lib.fea_plan_copy_crac(self._h, _ptr(row_ptr), _ptr(col_align)))
        return row_ptr, col_align

    def crac(self):
        row_ptr = np.empty(self.n_rows + 1, np.int64)
        col_align = np.empty(2 * self.n_runs + 2, np.int64)
        _check(self._lib.fea_plan_copy_crac(self._h, _ptr(row_ptr), _ptr(col_align)))
        return row_ptr, col_align

    def elements(self):
        out = np.empty(max(self.n_elements, 1), np.int64)
        _check(self._lib.fea_plan_copy_elements(self._h, _ptr(out)))
        return out[: self.n_elements]

    def greedy_colouring(self):
        col = np.empty(max(self.n_elements, 1), np.int32)
        nc = c_int32()
        _check(self._lib.fea_plan_greedy_colouring(self._h, _ptr(col), byref(nc)))
        return col[: self.n_elements], nc.value

    def jp_colouring(self, seed: int = 1):
        """Jones-Plassmann colouring on the device (valid; differs from the greedy one)."""
        col = np.empty(max(self.n_elements, 1), np.int32)
        nc = c_int32()
        _check(self._lib.fea_plan_jp_colouring(self._h, ctypes.c_uint64(seed), _ptr(col), byref(nc)))
        return col[: self.n_elements], nc.value

    def set_colouring(self, colour_of) -> None:
        col = np.ascontiguousarray(colour_of, dtype=np.int32)
        _check(self._lib.fea_plan_set_colouring(self._h, _ptr(col)))

    def missing_entry(self):
        e, r, c = c_int64(), c_int64(), c_int64()
        _check(self._lib.fea_plan_missing_entry(self._h, byref(e), byref(r), byref(c)))
        return None if e.value < 0 else (e.value, r.value, c.value)

    @property
    def last_launches(self) -> int:
        return int(self._lib.fea_plan_last_launches(self._h))

    # -- numeric phase ------------------------------------------------------
    def assemble(self, K, values=None, strategy: str = "sorted", accumulate: bool = False,
                 stream=None):
        """values (+)= assembled K. K: cuda float64 (E, m, m); values: cuda float64 (nnz,)."""
        import torch
        if values is None:
            values = torch.zeros(self.nnz, dtype=torch.float64, device=f"cuda:{self.device}")
            accumulate = False
        self._check_k(K)
        self._check_values(values)
        flags = (N.FEA_ACCUMULATE if accumulate else N.FEA_OVERWRITE) | _EXTRA_FLAGS.get(strategy, 0)
        _check(self._lib.fea_assemble(self._h, _ptr(K), STRATEGIES[strategy], _ptr(values), flags,
                                      _stream_ptr(stream, self.device)))
        return values

    def assemble_into(self, K, values_ptr: int, strategy: str = "sorted", accumulate: bool = False,
                      stream=None):
        """Assemble into a raw device address (e.g. this rank's row block inside the root's
        global values buffer, mapped with dist.PeerValues): the kernel's stores go to wherever
        the pointer lives, peer memory over NVLink included."""
        self._check_k(K)
        flags = (N.FEA_ACCUMULATE if accumulate else N.FEA_OVERWRITE) | _EXTRA_FLAGS.get(strategy, 0)
        _check(self._lib.fea_assemble(self._h, _ptr(K), STRATEGIES[strategy], c_void_p(values_ptr), flags,
                                      _stream_ptr(stream, self.device)))

    def assemble_seeded(self, seed: int, values=None, strategy: str = "sorted", accumulate: bool = False,
                        stream=None):
        """Fused supplier: assemble the seeded element matrices generated inside the kernel."""
        import torch
        if values is None:
            values = torch.zeros(self.nnz, dtype=torch.float64, device=f"cuda:{self.device}")
            accumulate = False
        self._check_values(values)
        flags = (N.FEA_ACCUMULATE if accumulate else N.FEA_OVERWRITE) | _EXTRA_FLAGS.get(strategy, 0)
        _check(self._lib.fea_assemble_seeded(self._h, ctypes.c_uint64(seed), STRATEGIES[strategy],
                                             _ptr(values), flags, _stream_ptr(stream, self.device)))
        return values

    def assemble_host(self, K_host, values_host=None, strategy: str = "sorted",
                      accumulate: bool = False, stream=None):
        """End-to-end form: host K in, host values out (H2D + assemble + D2H, synchronous)."""
        if values_host is None:
            values_host = np.zeros(self.nnz, np.float64)
            accumulate = False
        self._check_k(K_host, host=True)
        self._check_values(values_host, host=True)
        flags = (N.FEA_ACCUMULATE if accumulate else N.FEA_OVERWRITE) | _EXTRA_FLAGS.get(strategy, 0)
        _check(self._lib.fea_assemble_host(self._h, _ptr(K_host), STRATEGIES[strategy],
                                           _ptr(values_host), flags, _stream_ptr(stream, self.device)))
        return values_host

    def set_host_windows(self, n_windows: int) -> None:
        """Pipeline depth of assemble_host (0 = automatic; see fea_plan_set_host_windows)."""
        _check(self._lib.fea_plan_set_host_windows(self._h, int(n_windows)))

    def assemble_host_batch(self, K_hosts, values_hosts, strategy: str = "sorted",
                            accumulate: bool = False, stream=None):
        """Pipelined repeated end-to-end assemblies: K_hosts[i] (host) -> values_hosts[i] (host).
        Step i's K upload overlaps step i-1's kernel and values download (pinned memory)."""
        n = len(K_hosts)
        assert len(values_hosts) == n
        for k, v in zip(K_hosts, values_hosts):
            self._check_k(k, host=True)
            self._check_values(v, host=True)
        kp = (c_void_p * max(n, 1))(*[_ptr(k).value for k in K_hosts])
        vp = (c_void_p * max(n, 1))(*[_ptr(v).value for v in values_hosts])
        flags = (N.FEA_ACCUMULATE if accumulate else N.FEA_OVERWRITE) | _EXTRA_FLAGS.get(strategy, 0)
        _check(self._lib.fea_assemble_host_batch(self._h, kp, STRATEGIES[strategy], vp, n, flags,
                                                 _stream_ptr(stream, self.device)))
        return values_hosts

    def spmv(self, values, x, y=None, stream=None):
        """y = A x with the plan's node-block layout (device tensors; x over global columns)."""
        import torch
        if y is None:
            y = torch.empty(self.n_rows, dtype=torch.float64, device=values.device)
        _check(self._lib.fea_plan_spmv(self._h, _ptr(values), _ptr(x), _ptr(y), _stream_ptr(stream, self.device)))
        return y

    def close(self) -> None:
        if self._h and self._h.value:
            self._lib.fea_plan_destroy(self._h)
            self._h = c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def fill_seeded_k(n: int, m: int, seed: int, elem_ids=None, device: int = 0, out=None, stream=None):
    """Seeded symmetric U[-1,1) element matrices on the device (the counter-hash supplier)."""
    import torch
    if out is None:
        out = torch.empty((n, m, m), dtype=torch.float64, device=f"cuda:{device}")
    ids = None
    if elem_ids is not None:
        ids = torch.as_tensor(elem_ids, dtype=torch.int64, device=out.device).contiguous()
    _check(N.lib().fea_fill_seeded_k(_ptr(out), n, m, ctypes.c_uint64(seed), _ptr(ids),
                                     _stream_ptr(stream, out.device.index)))
    if ids is not None:
        torch.cuda.current_stream(out.device).synchronize()
    return out


def exclusive_sum(x, out=None, stream=None):
    """Exclusive prefix sum of a device int64 tensor (the symbolic phase's own scan, csrc/prims.cu)."""
    import torch
    if x.dtype != torch.int64 or not x.is_cuda or not x.is_contiguous():
        raise ValueError("exclusive_sum takes a contiguous CUDA int64 tensor")
    if out is None:
        out = torch.empty_like(x)
    _check(N.lib().fea_exclusive_sum_i64(_ptr(x), _ptr(out), x.numel(), _stream_ptr(stream, x.device.index)))
    return out


def sort_pairs(keys, vals, begin_bit: int = 0, end_bit: int = 32, stream=None):
    """Stable LSD radix sort of (uint32-valued keys, int32 vals) device pairs by key bits
    [begin_bit, end_bit) (csrc/prims.cu). keys: int32/uint32-width CUDA tensor (bit pattern)."""
    import torch
    if keys.element_size() != 4 or vals.dtype != torch.int32 or not keys.is_cuda or keys.numel() != vals.numel():
        raise ValueError("sort_pairs takes 4-byte CUDA keys and int32 values of equal length")
    keys, vals = keys.contiguous(), vals.contiguous()
    ko, vo = torch.empty_like(keys), torch.empty_like(vals)
    _check(N.lib().fea_sort_pairs_u32(_ptr(keys), _ptr(ko), _ptr(vals), _ptr(vo), keys.numel(), begin_bit,
                                      end_bit, _stream_ptr(stream, keys.device.index)))
    return ko, vo


def spmv_csr(row_ptr, cols, values, x, y=None, stream=None):
    """y = A x over device CSR arrays (int64 row_ptr/cols, fp64 values/x)."""
    import torch
    n = row_ptr.numel() - 1
    if y is None:
        y = torch.empty(n, dtype=torch.float64, device=values.device)
    _check(N.lib().fea_spmv_csr(_ptr(row_ptr), _ptr(cols), _ptr(values), n, _ptr(x), _ptr(y),
                                _stream_ptr(stream, values.device.index)))
    return y


def spmv_crac(crac_ptr, col_align, values, x, y=None, stream=None):
    """y = A x over device CRAC arrays (row_ptr in col_align entry units, col_align pairs)."""
    import torch
    n = crac_ptr.numel() - 1
    if y is None:
        y = torch.empty(n, dtype=torch.float64, device=values.device)
    _check(N.lib().fea_spmv_crac(_ptr(crac_ptr), _ptr(col_align), _ptr(values), n, _ptr(x), _ptr(y),
                                 _stream_ptr(stream, values.device.index)))
    return y
