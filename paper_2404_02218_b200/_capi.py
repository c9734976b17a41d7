"""ctypes mirror of include/hg/hg.h (the C-ABI of libhalogen_b200.so).

The library is built in-tree (``make -C paper_2404_02218_b200``) into
``paper_2404_02218_b200/lib/libhalogen_b200.so``.  There is no CPU fallback: if the library
is missing or the GPU path fails, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

HG_MAX_RANK = 3
HG_MAX_FIELDS = 16
HG_MAX_RESULTS = 8
HG_MAX_OPS = 4096
HG_MAX_APPLIES = 32
HG_MAX_TEMPS = 64
HG_MAX_STORES = 16

HG_OK, HG_EINVAL, HG_EUNSUPPORTED, HG_ECUDA, HG_ETRAP, HG_ENOMEM, HG_ESTATE = range(7)
HG_F32, HG_F64 = 1, 2
HG_TRANSPORT_P2P, HG_TRANSPORT_NCCL = 0, 1
HG_NCCL_ID_BYTES = 128
HG_OP_ACCESS, HG_OP_CONST, HG_OP_ADD, HG_OP_SUB, HG_OP_MUL, HG_OP_DIV = 1, 2, 3, 4, 5, 6

i64x3 = C.c_int64 * HG_MAX_RANK


class HgOp(C.Structure):
    _fields_ = [("code", C.c_int32), ("a", C.c_int32), ("b", C.c_int32),
                ("operand", C.c_int32), ("off", i64x3), ("bits", C.c_uint64)]


class HgDmpOpts(C.Structure):
    _fields_ = [("transport", C.c_int), ("nranks", C.c_int),
                ("nccl_id", C.c_ubyte * HG_NCCL_ID_BYTES), ("timeout_s", C.c_double),
                ("depth", C.c_int)]


class HgBounds(C.Structure):
    _fields_ = [("lb", i64x3), ("ub", i64x3)]


class HgApply(C.Structure):
    _fields_ = [("noperands", C.c_int32), ("operand", C.c_int32 * HG_MAX_FIELDS),
                ("op_begin", C.c_int32), ("nops", C.c_int32), ("nresults", C.c_int32),
                ("result_op", C.c_int32 * HG_MAX_RESULTS),
                ("result_temp", C.c_int32 * HG_MAX_RESULTS), ("domain", HgBounds)]


class HgProgram(C.Structure):
    _fields_ = [
        ("rank", C.c_int32), ("dtype", C.c_int32), ("nfields", C.c_int32),
        ("fields", HgBounds * HG_MAX_FIELDS),
        ("noperands", C.c_int32), ("operand_field", C.c_int32 * HG_MAX_FIELDS),
        ("nops", C.c_int32), ("ops", C.POINTER(HgOp)),
        ("nresults", C.c_int32), ("result_op", C.c_int32 * HG_MAX_RESULTS),
        ("store_field", C.c_int32 * HG_MAX_RESULTS), ("store", HgBounds * HG_MAX_RESULTS),
        ("ngroups", C.c_int32), ("group_len", C.c_int32 * HG_MAX_FIELDS),
        ("groups", C.c_int32 * HG_MAX_FIELDS),
        ("napplies", C.c_int32), ("applies", C.POINTER(HgApply)), ("ntemps", C.c_int32),
        ("nstores", C.c_int32), ("mstore_temp", C.c_int32 * HG_MAX_STORES),
        ("mstore_field", C.c_int32 * HG_MAX_STORES), ("mstore", HgBounds * HG_MAX_STORES),
    ]


class HgExchange(C.Structure):
    _fields_ = [("at", i64x3), ("size", i64x3), ("offset", i64x3), ("to", i64x3)]


class HgSwap(C.Structure):
    _fields_ = [("field", C.c_int32), ("nexchanges", C.c_int32),
                ("ex", HgExchange * (2 * HG_MAX_RANK))]


class HgDecomp(C.Structure):
    _fields_ = [("ndim", C.c_int32), ("grid", i64x3), ("core", i64x3),
                ("nswaps", C.c_int32), ("swaps", HgSwap * HG_MAX_FIELDS)]


class HgLayout(C.Structure):
    _fields_ = [("rank", C.c_int32), ("elem_bytes", C.c_int32), ("shape", i64x3),
                ("lb", i64x3), ("pitch", C.c_int64), ("col0", C.c_int64), ("rows", C.c_int64),
                ("device_ptr", C.c_void_p)]


LIB_PATH = os.environ.get("HG_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                    "lib", "libhalogen_b200.so")
_lib = None


class HgError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"hg status {status}: {msg}")
        self.status = status


def lib() -> C.CDLL:
    """Load the in-tree library; raise (never fall back) when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                           f"or `make -C paper_2404_02218_b200`")
    L = C.CDLL(LIB_PATH)
    P, V, I32, I64, SZ = C.POINTER, C.c_void_p, C.c_int32, C.c_int64, C.c_size_t
    sig = {
        "hg_last_error": (C.c_char_p, []),
        "hg_version": (C.c_int, []),
        "hg_device_count": (C.c_int, [P(C.c_int)]),
        "hg_init_value": (C.c_double, [C.c_int, C.c_int, P(I64)]),
        "hg_fingerprint": (C.c_uint64, [V, SZ]),
        "hg_binding_after": (C.c_int, [C.c_int, P(I32), P(I32), C.c_int, I64, P(I32)]),
        "hg_gpts_per_sec": (C.c_double, [I64, I64, C.c_double]),
        "hg_rank_from_coord": (I64, [C.c_int, P(I64), P(I64)]),
        "hg_coord_from_rank": (None, [C.c_int, I64, P(I64), P(I64)]),
        "hg_neighbor_rank": (I64, [C.c_int, I64, P(I64), P(I64)]),
        "hg_local_interval": (None, [I64, I64, I64, P(I64), P(I64)]),
        "hg_exchanges": (C.c_int, [C.c_int, P(I64), P(I64), P(I64), P(I64), P(I64),
                                   P(HgExchange), C.c_int]),
        "hg_build_kernel_program": (C.c_int, [C.c_char_p, C.c_int, I64, C.c_int, C.c_int,
                                              P(HgProgram), P(HgOp), C.c_int]),
        "hg_program_match": (C.c_int, [P(HgProgram), C.c_char_p, SZ]),
        "hg_apply_compile": (C.c_int, [P(HgProgram), C.c_char_p, SZ, P(SZ)]),
        "hg_fuse_applies": (C.c_int, [P(HgProgram), P(HgProgram), P(HgOp), C.c_int]),
        "hg_parse_program": (C.c_int, [C.c_char_p, P(HgProgram), P(HgOp), C.c_int, P(HgApply),
                                       C.c_int, P(HgDecomp), P(C.c_int), C.c_char_p, SZ]),
        "hg_decompose_program_deep": (C.c_int, [P(HgProgram), C.c_int, P(I64), C.c_int,
                                                P(HgProgram), P(HgDecomp)]),
        "hg_decompose_program": (C.c_int, [P(HgProgram), C.c_int, P(I64), P(HgProgram),
                                           P(HgDecomp)]),
        "hg_plan_create": (C.c_int, [P(HgProgram), C.c_int, P(V)]),
        "hg_plan_destroy": (C.c_int, [V]),
        "hg_plan_kernel_name": (C.c_int, [V, C.c_char_p, SZ]),
        "hg_plan_layout": (C.c_int, [V, C.c_int, P(HgLayout)]),
        "hg_plan_init_fields": (C.c_int, [V, P(I64), V]),
        "hg_plan_upload": (C.c_int, [V, C.c_int, V, SZ, V]),
        "hg_plan_upload_live": (C.c_int, [V, C.c_int, V, SZ, V]),
        "hg_plan_download": (C.c_int, [V, C.c_int, V, SZ, V]),
        "hg_plan_run": (C.c_int, [V, I64, V]),
        "hg_plan_binding": (C.c_int, [V, P(I32), P(I64)]),
        "hg_plan_reset_binding": (C.c_int, [V]),
        "hg_plan_pack": (C.c_int, [V, C.c_int, P(I64), P(I64), V, V]),
        "hg_plan_unpack": (C.c_int, [V, C.c_int, P(I64), P(I64), V, V]),
        "hg_plan_launch_count": (I64, [V]),
        "hg_plan_synchronize": (C.c_int, [V]),
        "hg_plan_check_guards": (C.c_int, [V]),
        "hg_plan_bind": (C.c_int, [V, C.c_int, V, SZ]),
        "hg_plan_set_tuning": (C.c_int, [V, C.c_int, C.c_int]),
        "hg_dmp_create": (C.c_int, [V, P(HgDecomp), I64, P(V)]),
        "hg_dmp_create_ex": (C.c_int, [V, P(HgDecomp), I64, P(HgDmpOpts), P(V)]),
        "hg_nccl_unique_id": (C.c_int, [V]),
        "hg_dmp_status": (C.c_int, [V]),
        "hg_dmp_set_timeout": (C.c_int, [V, C.c_double]),
        "hg_dmp_destroy": (C.c_int, [V]),
        "hg_dmp_ipc_export": (C.c_int, [V, V, SZ, P(SZ)]),
        "hg_dmp_ipc_import": (C.c_int, [V, I64, V, SZ]),
        "hg_dmp_run": (C.c_int, [V, I64, V]),
        "hg_sim_connect": (C.c_int, [P(V), C.c_int]),
        "hg_sim_run": (C.c_int, [P(V), C.c_int, I64, P(V)]),
        "hg_dmp_bytes_exchanged": (I64, [V]),
        "hg_dmp_invalidate": (C.c_int, [V]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(status: int) -> None:
    if status != HG_OK:
        msg = lib().hg_last_error()
        raise HgError(status, msg.decode() if msg else "")


def exported_symbols() -> list[str]:
    """Names declared in include/hg/hg.h (used by the CPU symbol-export test)."""
    here = os.path.dirname(os.path.abspath(__file__))
    hdr = os.path.join(here, "..", "include", "hg", "hg.h")
    import re
    names = []
    with open(hdr) as f:
        for line in f:
            m = re.match(r"^\s*[A-Za-z_][\w \*]*?\b(hg_\w+)\s*\(", line)
            if m:
                names.append(m.group(1))
    return names
