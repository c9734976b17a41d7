"""halogen-b200: B200-native stencil time stepping + dmp halo swap (arXiv 2404.02218 path).

Python host glue over the C-ABI of ``lib/libhalogen_b200.so`` (include/hg/hg.h).  The names
mirror the reference's C++ API in /root/reference/proj/core (exec::buildKernel,
exec::initialFields, exec::runSerialStencil, exec::bindingAfter, ir::dmp::*, exec::simulate);
the compute always runs in the sm_100a kernels -- there is no CPU fallback in this package.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field as dc_field
from typing import List, Optional, Sequence

import numpy as np

import os

from . import _capi as capi
from ._capi import HgDecomp, HgError, HgExchange, HgLayout, HgOp, HgProgram, check, lib  # noqa: F401

__all__ = [
    "KernelSpec", "Program", "Buffer", "Plan", "Dmp", "build_kernel", "initial_fields",
    "init_value", "fill_init", "fingerprint", "binding_after", "run_serial_stencil",
    "rank_from_coord", "coord_from_rank", "neighbor_rank", "local_interval", "exchanges",
    "simulate", "gpts_per_sec", "csv_header", "csv_row",
]

_I64 = C.c_int64
_DT = {capi.HG_F32: np.float32, capi.HG_F64: np.float64}


def _i64(v: Sequence[int]):
    return (_I64 * max(len(v), 1))(*v)


# ---- Buffer: the host field (exec::Buffer, buffer.hpp:25-57) --------------------------------
@dataclass
class Buffer:
    """Row-major host storage with the logical lower bound of its field type."""
    data: np.ndarray          # shape == alloc shape, halo included, C order
    lb: List[int]

    @staticmethod
    def for_bounds(dtype, lb: Sequence[int], ub: Sequence[int]) -> "Buffer":
        shape = [u - l for l, u in zip(lb, ub)]
        return Buffer(np.zeros(shape, dtype=dtype), list(lb))

    @property
    def shape(self):
        return list(self.data.shape)

    def clone(self) -> "Buffer":
        return Buffer(self.data.copy(), list(self.lb))

    def fingerprint(self) -> int:
        return fingerprint(self.data)


# ---- host algorithms ----------------------------------------------------------------------
def init_value(field_idx: int, coord: Sequence[int]) -> float:
    return lib().hg_init_value(field_idx, len(coord), _i64(coord))


def fingerprint(arr: np.ndarray) -> int:
    a = np.ascontiguousarray(arr)
    return int(lib().hg_fingerprint(a.ctypes.data_as(C.c_void_p), a.nbytes))


def binding_after(groups: Sequence[Sequence[int]], num_args: int, steps: int) -> List[int]:
    glen = (C.c_int32 * max(len(groups), 1))(*[len(g) for g in groups])
    flat = [i for g in groups for i in g]
    gg = (C.c_int32 * max(len(flat), 1))(*flat)
    out = (C.c_int32 * max(num_args, 1))()
    check(lib().hg_binding_after(len(groups), glen, gg, num_args, steps, out))
    return list(out[:num_args])


def gpts_per_sec(core_points: int, steps: int, seconds: float) -> float:
    return lib().hg_gpts_per_sec(core_points, steps, seconds)


def csv_header() -> str:
    return "label,core_points,steps,seconds,gpts_per_s"  # throughput.cpp:25-27


def csv_row(label: str, core_points: int, steps: int, seconds: float) -> str:
    return (f"{label},{core_points},{steps},{seconds:.17g},"
            f"{gpts_per_sec(core_points, steps, seconds):.17g}")


def rank_from_coord(coord: Sequence[int], grid: Sequence[int]) -> int:
    return lib().hg_rank_from_coord(len(grid), _i64(coord), _i64(grid))


def coord_from_rank(rank: int, grid: Sequence[int]) -> List[int]:
    out = (_I64 * 3)()
    lib().hg_coord_from_rank(len(grid), rank, _i64(grid), out)
    return list(out[:len(grid)])


def neighbor_rank(rank: int, direction: Sequence[int], grid: Sequence[int]) -> int:
    return lib().hg_neighbor_rank(len(grid), rank, _i64(direction), _i64(grid))


def local_interval(extent: int, parts: int, part: int):
    lb, ub = _I64(), _I64()
    lib().hg_local_interval(extent, parts, part, C.byref(lb), C.byref(ub))
    return lb.value, ub.value


def exchanges(core, below, above, grid=None, coord=None):
    n = len(core)
    out = (HgExchange * 6)()
    k = lib().hg_exchanges(n, _i64(core), _i64(below), _i64(above),
                           _i64(grid) if grid is not None else None,
                           _i64(coord) if coord is not None else None, out, 6)
    res = []
    for e in out[:k]:
        res.append({"at": list(e.at[:n]), "size": list(e.size[:n]),
                    "offset": list(e.offset[:n]), "to": list(e.to[:n])})
    return res


# ---- programs --------------------------------------------------------------------------------
@dataclass
class KernelSpec:
    """exec::KernelSpec (kernels.hpp:32-37) plus the element type of the retyped module."""
    kind: str = "heat"
    rank: int = 2
    extent: int = 64
    order: int = 2
    dtype: str = "f32"


class Program:
    """An hg_program plus the op storage it points into (the step function of a module)."""

    def __init__(self, prog: HgProgram, ops):
        self.prog = prog
        self.ops = ops
        self.applies = None
        self.prog.ops = C.cast(self.ops, C.POINTER(HgOp))

    @staticmethod
    def from_json(j) -> "Program":
        """A program descriptor serialised by tests/golden/make_golden.py (prog_json)."""
        p = HgProgram()
        ops = (HgOp * max(len(j["ops"]), 1))()
        r = j["rank"]
        p.rank, p.dtype, p.nfields = r, j["dtype"], j["nfields"]
        for i, (lb, ub) in enumerate(j["fields"]):
            for d in range(r):
                p.fields[i].lb[d], p.fields[i].ub[d] = lb[d], ub[d]
        loads = j["loads"] if "applies" in j else j["operand_field"]
        for i, f in enumerate(loads):
            p.operand_field[i] = f
        p.noperands = len(loads)
        for i, (code, a, b, operand, off, bits) in enumerate(j["ops"]):
            ops[i].code, ops[i].a, ops[i].b, ops[i].operand = code, a, b, operand
            for d in range(r):
                ops[i].off[d] = off[d]
            ops[i].bits = int(bits, 16)
        p.nops = len(j["ops"])
        if "applies" in j:  # multi-apply step
            aps = (capi.HgApply * max(len(j["applies"]), 1))()
            for a, A in enumerate(j["applies"]):
                aps[a].noperands = len(A["operands"])
                for o, x in enumerate(A["operands"]):
                    aps[a].operand[o] = x
                aps[a].op_begin, aps[a].nops = A["op_begin"], A["nops"]
                aps[a].nresults = len(A["result_op"])
                for k in range(aps[a].nresults):
                    aps[a].result_op[k] = A["result_op"][k]
                    aps[a].result_temp[k] = A["result_temp"][k]
                for d in range(r):
                    aps[a].domain.lb[d], aps[a].domain.ub[d] = A["domain"][0][d], A["domain"][1][d]
            p.napplies = len(j["applies"])
            p.ntemps = j["ntemps"]
            p.nstores = len(j["mstores"])
            for k, (t, f, lb, ub) in enumerate(j["mstores"]):
                p.mstore_temp[k], p.mstore_field[k] = t, f
                for d in range(r):
                    p.mstore[k].lb[d], p.mstore[k].ub[d] = lb[d], ub[d]
            p.ngroups = len(j["groups"])
            at = 0
            for g, grp in enumerate(j["groups"]):
                p.group_len[g] = len(grp)
                for x in grp:
                    p.groups[at] = x
                    at += 1
            prog = Program(p, ops)
            prog.applies = aps
            prog.prog.applies = C.cast(aps, C.POINTER(capi.HgApply))
            return prog
        p.nresults = len(j["result_op"])
        for k in range(p.nresults):
            p.result_op[k], p.store_field[k] = j["result_op"][k], j["store_field"][k]
            lb, ub = j["store"][k]
            for d in range(r):
                p.store[k].lb[d], p.store[k].ub[d] = lb[d], ub[d]
        p.ngroups = len(j["groups"])
        at = 0
        for g, grp in enumerate(j["groups"]):
            p.group_len[g] = len(grp)
            for x in grp:
                p.groups[at] = x
                at += 1
        return Program(p, ops)

    @staticmethod
    def parse(text: str):
        """Read `.xir` text (hg_parse_program).  Returns (Program, HgDecomp or None,
        dmp.reference text)."""
        ops = (HgOp * capi.HG_MAX_OPS)()
        aps = (capi.HgApply * capi.HG_MAX_APPLIES)()
        prog = HgProgram()
        dc = HgDecomp()
        dec = C.c_int()
        ref = C.create_string_buffer(1 << 20)
        check(lib().hg_parse_program(text.encode(), C.byref(prog), ops, capi.HG_MAX_OPS, aps,
                                     capi.HG_MAX_APPLIES, C.byref(dc), C.byref(dec), ref,
                                     1 << 20))
        out = Program(prog, ops)
        if prog.napplies > 0:
            out.applies = aps
            out.prog.applies = C.cast(aps, C.POINTER(capi.HgApply))
        return out, (dc if dec.value else None), ref.value.decode()

    @staticmethod
    def pw_advection(nz: int, ny: int, nx: int) -> "Program":
        """BASELINE config 4: the authored PW-advection program (programs/pw_advection.py),
        as exported by the reference's parser, resized to nz x ny x nx."""
        import json
        import os
        here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "programs",
                            "pw_advection.json")
        with open(here) as f:
            return Program.from_json(json.load(f)["program"]).with_extents([nz, ny, nx])

    @staticmethod
    def build(spec: KernelSpec) -> "Program":
        ops = (HgOp * capi.HG_MAX_OPS)()
        prog = HgProgram()
        dt = capi.HG_F32 if spec.dtype == "f32" else capi.HG_F64
        check(lib().hg_build_kernel_program(spec.kind.encode(), spec.rank, spec.extent,
                                            spec.order, dt, C.byref(prog), ops, capi.HG_MAX_OPS))
        return Program(prog, ops)

    @property
    def rank(self) -> int:
        return self.prog.rank

    @property
    def nfields(self) -> int:
        return self.prog.nfields

    @property
    def dtype(self):
        return _DT[self.prog.dtype]

    def field_bounds(self, i: int):
        b = self.prog.fields[i]
        return list(b.lb[:self.rank]), list(b.ub[:self.rank])

    def groups(self) -> List[List[int]]:
        out, at = [], 0
        for g in range(self.prog.ngroups):
            n = self.prog.group_len[g]
            out.append(list(self.prog.groups[at:at + n]))
            at += n
        return out

    def fuse_applies(self) -> "Program":
        """The multi-apply step as one single-apply program (hg_fuse_applies)."""
        ops = (HgOp * capi.HG_MAX_OPS)()
        out = HgProgram()
        check(lib().hg_fuse_applies(C.byref(self.prog), C.byref(out), ops, capi.HG_MAX_OPS))
        return Program(out, ops)

    def store_region(self, k: int = 0):
        """Stored region k (hg_bounds) of either program form."""
        return self.prog.mstore[k] if self.prog.napplies > 0 else self.prog.store[k]

    def core_points(self) -> int:
        s = self.store_region(0)
        n = 1
        for d in range(self.rank):
            n *= s.ub[d] - s.lb[d]
        return n

    def kernel_family(self) -> str:
        buf = C.create_string_buffer(128)
        check(lib().hg_program_match(C.byref(self.prog), buf, 128))
        return buf.value.decode()

    def decompose(self, grid: Sequence[int], depth: int = 1):
        """The decompose pass: returns (local program, HgDecomp).  depth > 1: halos and
        exchange boxes depth x as wide in the split dims (hg_decompose_program_deep), for a
        Dmp(..., depth=depth) that exchanges every `depth` steps."""
        local = HgProgram()
        dc = HgDecomp()
        aps = None
        if self.prog.napplies > 0:
            aps = (capi.HgApply * self.prog.napplies)()
            local.applies = C.cast(aps, C.POINTER(capi.HgApply))
        if depth > 1:
            check(lib().hg_decompose_program_deep(C.byref(self.prog), len(grid), _i64(grid),
                                                  depth, C.byref(local), C.byref(dc)))
        else:
            check(lib().hg_decompose_program(C.byref(self.prog), len(grid), _i64(grid),
                                             C.byref(local), C.byref(dc)))
        out = Program(local, self.ops)
        if aps is not None:
            out.applies = aps
        return out, dc

    def with_extents(self, extents: Sequence[int]) -> "Program":
        """The same step program over a non-cubic domain [0, extents) (buildKernel is cubic,
        kernels.cpp:155-158): store regions become [0, e) and every field keeps its halo."""
        p = HgProgram()
        C.pointer(p)[0] = self.prog
        r = p.rank
        for k in range(p.nresults):
            for d in range(r):
                p.store[k].lb[d] = 0
                p.store[k].ub[d] = extents[d]
        for i in range(p.nfields):
            for d in range(r):
                below = self.prog.store[0].lb[d] - self.prog.fields[i].lb[d]
                above = self.prog.fields[i].ub[d] - self.prog.store[0].ub[d]
                p.fields[i].lb[d] = -below
                p.fields[i].ub[d] = extents[d] + above
        return Program(p, self.ops)

    def op_list(self):
        return [self.ops[i] for i in range(self.prog.nops)]


def build_kernel(spec: KernelSpec) -> Program:
    return Program.build(spec)


def fill_init(buf: Buffer, field_idx: int, origin: Optional[Sequence[int]] = None) -> None:
    """exec::fillInit on the host (used for the reference-layout host buffers of tests)."""
    r = buf.data.ndim
    idx = np.indices(buf.data.shape).reshape(r, -1).T
    flat = buf.data.reshape(-1)
    org = list(origin) if origin is not None else [0] * r
    for k, raw in enumerate(idx):
        coord = [int(buf.lb[d] + raw[d] + org[d]) for d in range(r)]
        flat[k] = init_value(field_idx, coord)


def initial_fields(prog: Program) -> List[Buffer]:
    """exec::initialFields computed on the GPU (bit-identical), returned as host Buffers."""
    plan = Plan(prog)
    plan.init_fields()
    out = [Buffer(plan.download(i), prog.field_bounds(i)[0]) for i in range(prog.nfields)]
    plan.close()
    return out


# ---- plans -------------------------------------------------------------------------------------
_GUARDS = os.environ.get("HG_DEBUG_GUARDS", "") not in ("", "0")


class Plan:
    """Device-resident fields + compiled step (hg_plan)."""

    def __init__(self, prog: Program, device: int = 0):
        self.program = prog
        h = C.c_void_p()
        check(lib().hg_plan_create(C.byref(prog.prog), device, C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if self.h:
            h, self.h = self.h, None
            try:
                if _GUARDS:  # debug runs: no kernel may have written outside its buffers
                    check(lib().hg_plan_check_guards(h))
            finally:
                lib().hg_plan_destroy(h)

    def bind(self, b: int, device_ptr: int, nbytes: int):
        """hg_plan_bind: buffer b lives in caller memory (see layout(b) for its shape)."""
        check(lib().hg_plan_bind(self.h, b, C.c_void_p(device_ptr), nbytes))

    def check_guards(self):
        """HG_DEBUG_GUARDS=1 plans: raise HgError(HG_ETRAP) on an out-of-bounds write."""
        check(lib().hg_plan_check_guards(self.h))

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def kernel_name(self) -> str:
        buf = C.create_string_buffer(128)
        check(lib().hg_plan_kernel_name(self.h, buf, 128))
        return buf.value.decode()

    def layout(self, b: int) -> HgLayout:
        L = HgLayout()
        check(lib().hg_plan_layout(self.h, b, C.byref(L)))
        return L

    def init_fields(self, origin: Optional[Sequence[int]] = None, stream=None):
        check(lib().hg_plan_init_fields(self.h, _i64(origin) if origin is not None else None,
                                        stream))

    def upload(self, b: int, arr: np.ndarray, stream=None, live: bool = False):
        """live=True: skip the region the next step overwrites unread (hg_plan_upload_live);
        run at least one step before reading the buffer back."""
        a = np.ascontiguousarray(arr, dtype=self.program.dtype)
        fn = lib().hg_plan_upload_live if live else lib().hg_plan_upload
        check(fn(self.h, b, a.ctypes.data_as(C.c_void_p), a.nbytes, stream))

    def download(self, b: int, out: Optional[np.ndarray] = None, stream=None) -> np.ndarray:
        lo, hi = self.program.field_bounds(b)
        shape = [u - l for l, u in zip(lo, hi)]
        if out is None:
            out = np.empty(shape, dtype=self.program.dtype)
        check(lib().hg_plan_download(self.h, b, out.ctypes.data_as(C.c_void_p), out.nbytes,
                                     stream))
        return out

    def run(self, steps: int, stream=None):
        check(lib().hg_plan_run(self.h, steps, stream))

    def binding(self):
        perm = (C.c_int32 * capi.HG_MAX_FIELDS)()
        steps = _I64()
        check(lib().hg_plan_binding(self.h, perm, C.byref(steps)))
        return list(perm[:self.program.nfields]), steps.value

    def reset_binding(self):
        check(lib().hg_plan_reset_binding(self.h))

    def set_tuning(self, chunks: int = 0, boundary_last: bool = False):
        check(lib().hg_plan_set_tuning(self.h, chunks, 1 if boundary_last else 0))

    def launch_count(self) -> int:
        return int(lib().hg_plan_launch_count(self.h))

    def pack(self, b: int, at, size, dst_ptr: int, stream=None):
        check(lib().hg_plan_pack(self.h, b, _i64(at), _i64(size), C.c_void_p(dst_ptr), stream))

    def unpack(self, b: int, at, size, src_ptr: int, stream=None):
        check(lib().hg_plan_unpack(self.h, b, _i64(at), _i64(size), C.c_void_p(src_ptr),
                                   stream))


def run_serial_stencil(prog: Program, fields: List[Buffer], timesteps: int,
                       device: int = 0) -> List[Buffer]:
    """exec::runSerialStencil (serial.cpp:57-88) on the GPU.

    ``fields`` bind to the step arguments in order and are updated in place; the result is the
    final binding (result i is the buffer bound to argument i after the last rotation)."""
    if len(fields) != prog.nfields:
        raise ValueError("field count does not match the function")
    plan = Plan(prog, device)
    try:
        for i, f in enumerate(fields):
            plan.upload(i, f.data, live=timesteps > 0)
        plan.run(timesteps)
        for i, f in enumerate(fields):
            plan.download(i, f.data)
        perm, _ = plan.binding()
    finally:
        plan.close()
    return [fields[p] for p in perm]


# ---- dmp -------------------------------------------------------------------------------------
class Dmp:
    """One rank's halo-swap endpoint (hg_dmp) over a local plan.

    transport "p2p" (default): NVLink peer stores fused into the stencil kernel (connect the
    ranks with export()/import_peer(), see dist.connect).  transport "nccl": packed boxes over
    NCCL send/recv on a side stream; every rank passes the same `nccl_id` (nccl_unique_id() on
    one rank, shared by the host) and `nranks`.  timeout_s bounds every halo wait (0: the
    library default, < 0: forever)."""

    def __init__(self, plan: Plan, decomp: HgDecomp, rank: int, transport: str = "p2p",
                 nccl_id: Optional[bytes] = None, nranks: int = 0, timeout_s: float = 0.0,
                 depth: int = 1):
        self.plan = plan
        h = C.c_void_p()
        o = capi.HgDmpOpts()
        o.transport = capi.HG_TRANSPORT_NCCL if transport == "nccl" else capi.HG_TRANSPORT_P2P
        o.nranks = nranks
        o.timeout_s = timeout_s
        o.depth = depth
        if nccl_id is not None:
            C.memmove(o.nccl_id, nccl_id, capi.HG_NCCL_ID_BYTES)
        check(lib().hg_dmp_create_ex(plan.h, C.byref(decomp), rank, C.byref(o), C.byref(h)))
        self.h = h
        self.rank = rank
        self.transport = transport

    def close(self):
        if self.h:
            lib().hg_dmp_destroy(self.h)
            self.h = None

    def export(self) -> bytes:
        n = C.c_size_t()
        check(lib().hg_dmp_ipc_export(self.h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        check(lib().hg_dmp_ipc_export(self.h, buf, n.value, C.byref(n)))
        return buf.raw[:n.value]

    def import_peer(self, peer_rank: int, blob: bytes):
        b = C.create_string_buffer(blob, len(blob))
        check(lib().hg_dmp_ipc_import(self.h, peer_rank, b, len(blob)))

    def run(self, steps: int, stream=None):
        check(lib().hg_dmp_run(self.h, steps, stream))

    def status(self):
        """Wait for the queued work; raises HgError(HG_ETRAP) if a halo wait timed out."""
        check(lib().hg_dmp_status(self.h))

    def set_timeout(self, seconds: float):
        check(lib().hg_dmp_set_timeout(self.h, seconds))

    def bytes_exchanged(self) -> int:
        return int(lib().hg_dmp_bytes_exchanged(self.h))

    def invalidate(self):
        """Host data was uploaded: every halo is stale (collective across P2P ranks)."""
        check(lib().hg_dmp_invalidate(self.h))


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId through the library (for Dmp(..., transport="nccl"))."""
    buf = C.create_string_buffer(capi.HG_NCCL_ID_BYTES)
    check(lib().hg_nccl_unique_id(buf))
    return buf.raw


def simulate(prog: Program, grid: Sequence[int], global_init: List[Buffer], timesteps: int,
             devices: Optional[Sequence[int]] = None, depth: int = 1) -> List[Buffer]:
    """exec::simulate (simulator.cpp:1066-1203): decompose, scatter, run every rank on the
    GPU(s) of this process with device halo swaps, gather the cores.

    Result i = global field bound to slot i at the end, gathered over a copy of the initial
    global buffer of that slot's origin (so the global-boundary ring is the initial one).
    depth > 1: deep halos (exchange every `depth` steps, needs one rank per device)."""
    local, dc = prog.decompose(grid, depth=depth)
    nranks = int(np.prod(grid))
    ndev = lib_device_count()
    devs = list(devices) if devices is not None else [r % max(ndev, 1) for r in range(nranks)]
    plans, dmps = [], []
    try:
        for r in range(nranks):
            pl = Plan(local, devs[r])
            coord = coord_from_rank(r, grid)
            for f in range(prog.nfields):
                g = global_init[f]
                llo, lhi = local.field_bounds(f)
                lo = [llo[d] + coord[d] * dc.core[d] - g.lb[d] for d in range(prog.rank)]
                hi = [lhi[d] + coord[d] * dc.core[d] - g.lb[d] for d in range(prog.rank)]
                if all(lo[d] >= 0 and hi[d] <= g.data.shape[d] for d in range(prog.rank)):
                    sl = tuple(slice(lo[d], hi[d]) for d in range(prog.rank))
                    pl.upload(f, g.data[sl])       # scatterRank (simulator.cpp:995-1025)
                else:  # deep halos reach past the global ring: those cells are never read
                    a = np.zeros([hi[d] - lo[d] for d in range(prog.rank)], dtype=g.data.dtype)
                    src = tuple(slice(max(lo[d], 0), min(hi[d], g.data.shape[d]))
                                for d in range(prog.rank))
                    dst = tuple(slice(max(lo[d], 0) - lo[d], min(hi[d], g.data.shape[d]) - lo[d])
                                for d in range(prog.rank))
                    a[dst] = g.data[src]
                    pl.upload(f, a)
            plans.append(pl)
            dmps.append(Dmp(pl, dc, r, depth=depth))
        arr = (C.c_void_p * nranks)(*[d.h for d in dmps])
        check(lib().hg_sim_connect(arr, nranks))
        check(lib().hg_sim_run(arr, nranks, timesteps, None))
        perm, _ = plans[0].binding()
        out = [global_init[perm[i]].clone() for i in range(prog.nfields)]
        for r in range(nranks):                 # gatherRank (simulator.cpp:1027-1060)
            coord = coord_from_rank(r, grid)
            for i in range(prog.nfields):
                loc = plans[r].download(perm[i])
                llo, _ = local.field_bounds(perm[i])
                g = out[i]
                sr = local.store_region(0)
                src = tuple(slice(sr.lb[d] - llo[d], sr.ub[d] - llo[d]) for d in range(prog.rank))
                dst = tuple(slice(sr.lb[d] + coord[d] * dc.core[d] - g.lb[d],
                                  sr.ub[d] + coord[d] * dc.core[d] - g.lb[d])
                            for d in range(prog.rank))
                g.data[dst] = loc[src]
        return out
    finally:
        for d in dmps:
            d.close()
        for p in plans:
            p.close()


def lib_device_count() -> int:
    n = C.c_int()
    lib().hg_device_count(C.byref(n))
    return n.value
