"""Python access to the oracles (TEST INFRASTRUCTURE ONLY).

* ``Port``  -- oracle/libhg_oracle.so, the plain-C restatement of the reference algorithm
  (oracle/hg_oracle.c).  Built by ``make -C oracle port``; pinned against tests/golden/.
* ``Ref``   -- oracle/_ref/libhalogen_ref.so, the UNMODIFIED reference core compiled from
  /root/reference by ``make -C oracle ref`` (only where the reference exists; the built .so
  travels to the GPU box).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
import this module.  The product (paper_2404_02218_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import sys
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from paper_2404_02218_b200 import _capi as capi  # descriptor structs only  # noqa: E402

PORT_PATH = os.path.join(HERE, "libhg_oracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libhalogen_ref.so")


class OrBuf(C.Structure):
    _fields_ = [("rank", C.c_int), ("elem", C.c_int), ("shape", C.c_int64 * 3),
                ("lb", C.c_int64 * 3), ("data", C.c_void_p)]


def _orbuf(arr: np.ndarray, lb: Sequence[int]) -> OrBuf:
    assert arr.flags["C_CONTIGUOUS"]
    b = OrBuf()
    b.rank = arr.ndim
    b.elem = arr.itemsize
    for d in range(arr.ndim):
        b.shape[d] = arr.shape[d]
        b.lb[d] = lb[d]
    b.data = arr.ctypes.data
    return b


def _i64(v):
    return (C.c_int64 * max(len(v), 1))(*v)


class Port:
    """The C restatement (hg_oracle.c)."""

    def __init__(self, path: str = PORT_PATH):
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: make -C oracle port")
        L = C.CDLL(path)
        P = C.POINTER
        L.or_init_value.restype = C.c_double
        L.or_init_value.argtypes = [C.c_int, C.c_int, P(C.c_int64)]
        L.or_fill_init.argtypes = [P(OrBuf), C.c_int, P(C.c_int64)]
        L.or_fingerprint.restype = C.c_uint64
        L.or_fingerprint.argtypes = [P(OrBuf)]
        L.or_binding_after.argtypes = [C.c_int, P(C.c_int32), P(C.c_int32), C.c_int, C.c_int64,
                                       P(C.c_int32)]
        L.or_run.argtypes = [P(capi.HgProgram), P(P(OrBuf)), C.c_int64, P(C.c_int32), C.c_int]
        L.or_neighbor_rank.restype = C.c_int64
        L.or_neighbor_rank.argtypes = [C.c_int, C.c_int64, P(C.c_int64), P(C.c_int64)]
        L.or_exchanges.argtypes = [C.c_int, P(C.c_int64), P(C.c_int64), P(C.c_int64),
                                   P(C.c_int64), P(C.c_int64), P(capi.HgExchange), C.c_int]
        L.or_pack.argtypes = [P(OrBuf), P(C.c_int64), P(C.c_int64), C.c_void_p]
        L.or_unpack.argtypes = [P(OrBuf), P(C.c_int64), P(C.c_int64), C.c_void_p]
        L.or_simulate.argtypes = [P(capi.HgProgram), P(capi.HgDecomp), P(P(OrBuf)), C.c_int,
                                  C.c_int64, P(P(OrBuf)), C.c_int]
        L.or_simulate_rank_state.argtypes = [P(capi.HgProgram), P(capi.HgDecomp), P(P(OrBuf)),
                                             C.c_int, C.c_int64, C.c_int64, P(P(OrBuf)), C.c_int]
        L.or_last_error.restype = C.c_char_p
        self.L = L

    def _err(self, rc):
        if rc:
            raise RuntimeError("oracle: " + self.L.or_last_error().decode())

    def init_value(self, field: int, coord: Sequence[int]) -> float:
        return self.L.or_init_value(field, len(coord), _i64(coord))

    def fill(self, arr: np.ndarray, lb, field: int, origin=None) -> np.ndarray:
        b = _orbuf(arr, lb)
        self.L.or_fill_init(C.byref(b), field, _i64(origin) if origin is not None else None)
        return arr

    def initial_fields(self, prog) -> List[np.ndarray]:
        out = []
        for i in range(prog.nfields):
            lo, hi = prog.field_bounds(i)
            a = np.zeros([u - l for l, u in zip(lo, hi)], dtype=prog.dtype)
            self.fill(a, lo, i)
            out.append(a)
        return out

    def fingerprint(self, arr: np.ndarray) -> int:
        b = _orbuf(np.ascontiguousarray(arr), [0] * arr.ndim)
        return int(self.L.or_fingerprint(C.byref(b)))

    def run(self, prog, arrays: List[np.ndarray], T: int, nthreads: int = 0):
        """runSerialStencil on host arrays in place; returns the binding permutation."""
        bufs = [_orbuf(a, prog.field_bounds(i)[0]) for i, a in enumerate(arrays)]
        arr = (C.POINTER(OrBuf) * len(bufs))(*[C.pointer(b) for b in bufs])
        perm = (C.c_int32 * 16)()
        self._err(self.L.or_run(C.byref(prog.prog), arr, T, perm, nthreads or os.cpu_count()))
        return list(perm[:prog.nfields])

    def exchanges(self, core, below, above, grid=None, coord=None):
        n = len(core)
        out = (capi.HgExchange * 6)()
        k = self.L.or_exchanges(n, _i64(core), _i64(below), _i64(above),
                                _i64(grid) if grid is not None else None,
                                _i64(coord) if coord is not None else None, out, 6)
        return [{"at": list(e.at[:n]), "size": list(e.size[:n]), "offset": list(e.offset[:n]),
                 "to": list(e.to[:n])} for e in out[:k]]

    def pack(self, arr, lb, at, size) -> np.ndarray:
        out = np.empty(int(np.prod(size)), dtype=arr.dtype)
        self._err(self.L.or_pack(C.byref(_orbuf(arr, lb)), _i64(at), _i64(size),
                                 out.ctypes.data))
        return out

    def unpack(self, arr, lb, at, size, packed: np.ndarray):
        self._err(self.L.or_unpack(C.byref(_orbuf(arr, lb)), _i64(at), _i64(size),
                                   np.ascontiguousarray(packed).ctypes.data))

    def simulate(self, local_prog, decomp, global_arrays, global_lbs, T, nthreads=0):
        n = len(global_arrays)
        gb = [_orbuf(a, lb) for a, lb in zip(global_arrays, global_lbs)]
        outs = [np.empty_like(a) for a in global_arrays]
        ob = [_orbuf(a, lb) for a, lb in zip(outs, global_lbs)]
        ga = (C.POINTER(OrBuf) * n)(*[C.pointer(b) for b in gb])
        oa = (C.POINTER(OrBuf) * n)(*[C.pointer(b) for b in ob])
        self._err(self.L.or_simulate(C.byref(local_prog.prog), C.byref(decomp), ga, n, T, oa,
                                     nthreads or os.cpu_count()))
        return outs

    def simulate_rank_state(self, local_prog, decomp, global_arrays, global_lbs, T, rank,
                            nthreads=0):
        n = len(global_arrays)
        gb = [_orbuf(a, lb) for a, lb in zip(global_arrays, global_lbs)]
        outs = []
        for i in range(n):
            lo, hi = local_prog.field_bounds(i)
            outs.append(np.zeros([u - l for l, u in zip(lo, hi)], dtype=global_arrays[0].dtype))
        ob = [_orbuf(a, local_prog.field_bounds(i)[0]) for i, a in enumerate(outs)]
        ga = (C.POINTER(OrBuf) * n)(*[C.pointer(b) for b in gb])
        oa = (C.POINTER(OrBuf) * n)(*[C.pointer(b) for b in ob])
        self._err(self.L.or_simulate_rank_state(C.byref(local_prog.prog), C.byref(decomp), ga,
                                                n, T, rank, oa, nthreads or os.cpu_count()))
        return outs


class Ref:
    """The reference core itself (oracle/_ref/libhalogen_ref.so)."""

    def __init__(self, path: str = REF_PATH):
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: make -C oracle ref (needs /root/reference)")
        L = C.CDLL(path)
        V, P, LL = C.c_void_p, C.POINTER, C.c_longlong
        for name, res, args in [
            ("hr_last_error", C.c_char_p, []),
            ("hr_parse", V, [C.c_char_p]),
            ("hr_build_kernel", V, [C.c_char_p, C.c_int, LL, C.c_int, C.c_int]),
            ("hr_print", V, [V]),
            ("hr_free_str", None, [V]),
            ("hr_pipeline", V, [V, C.c_char_p]),
            ("hr_module_free", None, [V]),
            ("hr_initial_fields", V, [V]),
            ("hr_bufs_clone", V, [V]),
            ("hr_bufs_free", None, [V]),
            ("hr_bufs_count", C.c_int, [V]),
            ("hr_buf_info", C.c_int, [V, C.c_int, P(C.c_int), P(C.c_int), P(LL), P(LL)]),
            ("hr_buf_data", V, [V, C.c_int]),
            ("hr_fingerprint", C.c_ulonglong, [V, C.c_int]),
            ("hr_run_serial", V, [V, V, LL]),
            ("hr_time_serial", C.c_double, [V, V, LL]),
            ("hr_simulate", V, [V, V, LL, C.c_ulonglong]),
            ("hr_time_simulate", C.c_double, [V, V, LL]),
            ("hr_scatter_rank", V, [V, V, LL]),
            ("hr_init_value", C.c_double, [C.c_int, C.c_int, P(LL)]),
            ("hr_rank_from_coord", LL, [C.c_int, P(LL), P(LL)]),
            ("hr_coord_from_rank", None, [C.c_int, LL, P(LL), P(LL)]),
            ("hr_neighbor_rank", LL, [C.c_int, LL, P(LL), P(LL)]),
            ("hr_local_interval", None, [LL, LL, LL, P(LL), P(LL)]),
            ("hr_exchanges", C.c_int, [C.c_int, P(LL), P(LL), P(LL), P(LL), P(LL), P(LL),
                                       C.c_int]),
            ("hr_binding_after", None, [C.c_int, P(C.c_int), P(C.c_int), C.c_int, LL,
                                        P(C.c_int)]),
            ("hr_laplacian_weight", C.c_double, [C.c_int, LL]),
            ("hr_export_program", C.c_int, [V, P(capi.HgProgram), P(capi.HgOp), C.c_int,
                                            P(capi.HgDecomp), P(C.c_int), P(capi.HgApply),
                                            C.c_int]),
        ]:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        self.L = L

    def err(self):
        return self.L.hr_last_error().decode()

    def build(self, kind, rank, extent, order, f32=True):
        m = self.L.hr_build_kernel(kind.encode(), rank, extent, order, 1 if f32 else 0)
        if not m:
            raise RuntimeError(self.err())
        return m

    def parse(self, text: str):
        m = self.L.hr_parse(text.encode())
        if not m:
            raise RuntimeError(self.err())
        return m

    def print(self, mod) -> str:
        p = self.L.hr_print(mod)
        s = C.string_at(p).decode()
        self.L.hr_free_str(p)
        return s

    def pipeline(self, mod, pipe: str):
        m = self.L.hr_pipeline(mod, pipe.encode())
        if not m:
            raise RuntimeError(self.err())
        return m

    def bufs_to_numpy(self, bufs) -> List[tuple]:
        out = []
        for i in range(self.L.hr_bufs_count(bufs)):
            eb, rk = C.c_int(), C.c_int()
            shape, lb = (C.c_longlong * 3)(), (C.c_longlong * 3)()
            self.L.hr_buf_info(bufs, i, C.byref(eb), C.byref(rk), shape, lb)
            dt = np.float32 if eb.value == 4 else np.float64
            n = int(np.prod(shape[:rk.value]))
            ptr = self.L.hr_buf_data(bufs, i)
            a = np.ctypeslib.as_array((C.c_char * (n * eb.value)).from_address(ptr))
            out.append((a.view(dt).reshape(shape[:rk.value]).copy(), list(lb[:rk.value])))
        return out

    def export_program(self, mod):
        prog = capi.HgProgram()
        ops = (capi.HgOp * capi.HG_MAX_OPS)()
        applies = (capi.HgApply * capi.HG_MAX_APPLIES)()
        dc = capi.HgDecomp()
        dec = C.c_int()
        n = self.L.hr_export_program(mod, C.byref(prog), ops, capi.HG_MAX_OPS, C.byref(dc),
                                     C.byref(dec), applies, capi.HG_MAX_APPLIES)
        if n < 0:
            raise RuntimeError(self.err())
        prog._applies_keepalive = applies
        return prog, ops, (dc if dec.value else None)
