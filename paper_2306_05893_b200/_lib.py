"""ctypes binding of libtsb.so (include/tsb.h) plus the device-buffer helpers.

The CUDA path is the product: if the library or a GPU is missing, every
device entry point raises instead of falling back to a CPU implementation.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libtsb.so"

TSB_OK = 0
TSB_E_ASSEMBLY = 1
TSB_E_STALE_MAPPING = 2
TSB_E_SOLVER = 3
TSB_E_LIFECYCLE = 4
TSB_E_CUDA = 5
TSB_E_MODEL = 6
TSB_E_ARG = 7
TSB_E_PRECOND = 8

PRECOND_IDENTITY = 0
PRECOND_JACOBI = 1
PRECOND_LDLT = 2

c_i64 = C.c_int64
c_i32 = C.c_int32
c_vp = C.c_void_p


class AsmPlan(C.Structure):
    _fields_ = [
        ("n_nodes", c_i64), ("n_elems", c_i64), ("n_blocks", c_i64), ("nnz", c_i64),
        ("n_fixed_slots", c_i64),
        ("d_conn", c_vp), ("d_grads", c_vp), ("d_vol", c_vp), ("d_mass_share", c_vp),
        ("d_rest", c_vp), ("d_mass_diag", c_vp), ("d_gravity", c_vp), ("d_fixed_dof", c_vp),
        ("d_blk", c_vp), ("d_blk_list", c_vp), ("d_node_ptr", c_vp), ("d_node_list", c_vp),
        ("d_fixed_slots", c_vp), ("d_work", c_vp), ("d_flags", c_vp), ("d_gab", c_vp),
        ("d_blk_mirror", c_vp),
    ]


class AsmCoeffs(C.Structure):
    _fields_ = [
        ("lam", C.c_double), ("mu", C.c_double), ("h", C.c_double),
        ("rayleigh_stiffness", C.c_double), ("rayleigh_mass", C.c_double),
        ("cm", C.c_double), ("ck", C.c_double), ("law", c_i32), ("want_matrix", c_i32),
    ]


class LdltDesc(C.Structure):
    _fields_ = [
        ("n", c_i64), ("n_blocks", c_i64), ("n_items_lower", c_i64), ("n_items_upper", c_i64),
        ("max_m", c_i32), ("max_v", c_i32), ("max_cb", c_i32), ("grid", c_i32),
        ("d_blocks", c_vp), ("d_items_lower", c_vp), ("d_items_upper", c_vp),
        ("d_tiles_lower", c_vp), ("d_tiles_upper", c_vp), ("d_g", c_vp), ("d_gt", c_vp),
        ("d_anc", c_vp), ("d_cslot", c_vp), ("d_cin_ptr", c_vp), ("d_d", c_vp), ("d_perm", c_vp),
        ("d_cbuf", c_vp), ("d_x", c_vp), ("d_y", c_vp),
        ("d_cnt_l", c_vp), ("d_ready_l", c_vp), ("d_done_u", c_vp), ("d_pad", c_vp),
        ("d_part_lower", c_vp), ("d_part_upper", c_vp), ("d_tcnt_lower", c_vp), ("d_tcnt_upper", c_vp),
        ("n_tiles_lower", c_i64), ("n_tiles_upper", c_i64), ("d_ext_rows", c_vp), ("n_ext", c_i64),
        ("d_ctl", c_vp),
        ("d_trace_lower", c_vp), ("d_trace_upper", c_vp), ("d_rin", c_vp),
    ]


class RefactorDesc(C.Structure):
    _fields_ = [
        ("n_fronts", c_i64), ("n_prog", c_i64), ("h_prog", c_vp), ("d_fronts", c_vp), ("d_lists", c_vp),
        ("d_sc_src", c_vp), ("d_sc_dst", c_vp), ("d_pairs", c_vp), ("d_tp", c_vp),
        ("d_tiles_lower", c_vp), ("d_tiles_upper", c_vp), ("d_tile_blk_lower", c_vp), ("d_tile_blk_upper", c_vp),
        ("n_tiles_lower", c_i64), ("n_tiles_upper", c_i64),
        ("d_ws", c_vp), ("d_wb", c_vp), ("d_inv", c_vp), ("ws_size", c_i64), ("wb_size", c_i64), ("d_ctl", c_vp),
    ]


class PatternDesc(C.Structure):
    _fields_ = [
        ("n_nodes", c_i64), ("n_elems", c_i64), ("d_conn", c_vp), ("d_pinned", c_vp), ("d_tmp", c_vp),
        ("d_sums", c_vp), ("d_node_ptr", c_vp), ("d_node_list", c_vp), ("d_cand", c_vp), ("d_nbr", c_vp),
        ("d_blk_ptr", c_vp), ("d_row_base", c_vp), ("n_blocks", c_i64), ("nnz", c_i64), ("n_contrib", c_i64),
        ("d_ccount", c_vp), ("d_cptr", c_vp), ("d_row_ptr", c_vp), ("d_col_ind", c_vp), ("d_blk", c_vp),
        ("d_blk_list", c_vp),
    ]


class Report(C.Structure):
    _fields_ = [
        ("iterations", c_i64), ("final_residual", C.c_double), ("converged", c_i32),
        ("status", c_i32), ("zero_diag_row", c_i64),
    ]


# every symbol include/tsb.h declares, with its ctypes signature
_SIGNATURES = {
    "tsb_abi_version": (C.c_int, []),
    "tsb_last_error": (C.c_int, [C.c_char_p, C.c_size_t]),
    "tsb_launch_count": (c_i64, []),
    "tsb_struct_size": (c_i64, [c_i32]),
    "tsb_spmv": (C.c_int, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "tsb_csr_diagonal": (C.c_int, [c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "tsb_compress": (C.c_int, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "tsb_assembly_setup": (C.c_int, [C.POINTER(AsmPlan), c_vp]),
    "tsb_assemble_corot": (C.c_int, [C.POINTER(AsmPlan), C.POINTER(AsmCoeffs), c_vp, c_vp, c_vp,
                                     c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "tsb_element_blocks": (C.c_int, [C.POINTER(AsmPlan), C.POINTER(AsmCoeffs), c_vp, c_vp, c_vp]),
    "tsb_advance": (C.c_int, [c_i64, c_vp, c_vp, c_vp, c_vp, C.c_double, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "tsb_ldlt_create": (C.c_int, [C.POINTER(LdltDesc), C.POINTER(c_vp)]),
    "tsb_ldlt_destroy": (C.c_int, [c_vp]),
    "tsb_ldlt_lower": (C.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "tsb_ldlt_upper": (C.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "tsb_ldlt_apply": (C.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "tsb_ldlt_lower_multi": (C.c_int, [c_vp, c_i32, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp]),
    "tsb_ldlt_lower_ext": (C.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "tsb_ldlt_upper_scaled": (C.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "tsb_ldlt_external_sums": (C.c_int, [c_vp, c_vp, c_vp]),
    "tsb_wdot": (C.c_int, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "tsb_pcg_update": (C.c_int, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "tsb_pcg_direction": (C.c_int, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "tsb_pcg_check": (C.c_int, [c_vp, C.c_double, C.c_double, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "tsb_peer_allreduce": (C.c_int, [c_i64, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp]),
    "tsb_spmv_peer": (C.c_int, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i32, c_i32, c_vp, c_vp, c_vp,
                                c_i64, c_i64, c_vp, c_vp]),
    "tsb_ldlt_external_sums_peer": (C.c_int, [c_vp, c_vp, c_i64, c_i32, c_i32, c_vp, c_vp, c_vp, c_i64, c_i64,
                                              c_vp, c_vp]),
    "tsb_gather_rows": (C.c_int, [c_i64, c_vp, c_vp, c_vp, c_vp]),
    "tsb_scatter_rows": (C.c_int, [c_i64, c_vp, c_vp, c_vp, c_vp]),
    "tsb_pcg_create": (C.c_int, [c_i64, C.POINTER(c_vp)]),
    "tsb_pcg_destroy": (C.c_int, [c_vp]),
    "tsb_pcg_solve": (C.c_int, [c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_vp,
                                c_vp, C.c_double, c_i64, C.POINTER(Report), c_vp]),
    "tsb_pcg_report": (C.c_int, [c_vp, C.POINTER(Report), c_vp]),
    "tsb_pcg_phase_times": (C.c_int, [c_vp, c_vp, c_vp]),
    "tsb_plane_contacts": (C.c_int, [c_i64, c_vp, C.c_double, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "tsb_contact_rhs": (C.c_int, [c_i64, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "tsb_gram_scratch": (c_i64, [c_i64, c_i64]),
    "tsb_gram": (C.c_int, [c_i64, c_i64, c_vp, c_vp, C.c_double, c_vp, c_vp, c_vp]),
    "tsb_compliance_from_columns": (C.c_int, [c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, C.c_double, c_vp, c_vp]),
    "tsb_pgs": (C.c_int, [c_i64, c_vp, c_vp, c_vp, C.c_double, c_i32, c_vp, c_vp, c_vp]),
    "tsb_gemv_cols": (C.c_int, [c_i64, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "tsb_contact_correct": (C.c_int, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "tsb_pattern_count": (C.c_int, [C.POINTER(PatternDesc), c_vp]),
    "tsb_pattern_fill": (C.c_int, [C.POINTER(PatternDesc), c_vp]),
    "tsb_refactor_create": (C.c_int, [C.POINTER(RefactorDesc), C.POINTER(c_vp)]),
    "tsb_refactor_destroy": (C.c_int, [c_vp]),
    "tsb_refactor_run": (C.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "tsb_nested_dissection": (C.c_int, [c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp,
                                        c_vp, c_vp, c_vp]),
}

ABI_VERSION = 3
_lib = None
_lock = threading.Lock()


class NativeLibraryError(RuntimeError):
    """libtsb.so is missing or incompatible (build it with __graft_entry__.build())."""


def load() -> C.CDLL:
    """Load libtsb.so (raises NativeLibraryError; there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = Path(os.environ.get("TSB_LIB", LIB_PATH))
        if not path.exists():
            raise NativeLibraryError(
                f"{path} not found: build it with `python -m paper_2306_05893_b200.build`"
            )
        lib = C.CDLL(str(path))
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.tsb_abi_version() != ABI_VERSION:
            raise NativeLibraryError("libtsb ABI version mismatch")
        for k, st in enumerate((AsmPlan, AsmCoeffs, None, LdltDesc, Report, None, None, None, RefactorDesc, PatternDesc)):
            if st is not None and lib.tsb_struct_size(k) != C.sizeof(st):
                raise NativeLibraryError(f"libtsb struct layout mismatch: {st.__name__}")
        _lib = lib
    return _lib


def exported_symbols():
    return list(_SIGNATURES)


def last_error() -> str:
    buf = C.create_string_buffer(4096)
    load().tsb_last_error(buf, len(buf))
    return buf.value.decode(errors="replace")


def check(status: int, what: str = ""):
    """Map a tsb status code to the reference's exception types."""
    if status == TSB_OK:
        return
    msg = last_error() or what
    from . import assembly, krylov, models, ndprecond  # local: avoid import cycles

    exc = {
        TSB_E_ASSEMBLY: assembly.AssemblyError,
        TSB_E_STALE_MAPPING: assembly.StaleMappingError,
        TSB_E_SOLVER: krylov.SolverError,
        TSB_E_LIFECYCLE: ndprecond.LifecycleError,
        TSB_E_MODEL: models.ModelError,
        TSB_E_PRECOND: ndprecond.PrecondError,
        TSB_E_ARG: ValueError,
    }.get(status, RuntimeError)
    raise exc(f"{what}: {msg}" if what else msg)


def launch_count() -> int:
    return int(load().tsb_launch_count())


# ---------------------------------------------------------------------------
# torch buffer helpers (torch is used for device memory and streams only)
# ---------------------------------------------------------------------------

def torch():
    import torch as _t

    return _t


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise NativeLibraryError("the B200 path needs a CUDA device; no CPU fallback exists")
    load()
    return t


def is_cuda_ready() -> bool:
    try:
        return bool(torch().cuda.is_available()) and load() is not None
    except Exception:
        return False


def stream_ptr(stream=None) -> int:
    t = torch()
    s = stream if stream is not None else t.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(tensor) -> int | None:
    return None if tensor is None else int(tensor.data_ptr())


def to_device(a, dtype=None, device="cuda"):
    """numpy/torch -> contiguous CUDA tensor (no copy if already there)."""
    t = torch()
    if isinstance(a, t.Tensor):
        out = a.to(device=device, dtype=dtype) if dtype is not None else a.to(device=device)
        return out.contiguous()
    arr = np.ascontiguousarray(a)
    if dtype is not None:
        arr = arr.astype(np.dtype(str(dtype).replace("torch.", "")), copy=False)
    if not arr.flags.writeable:  # read-only inputs (e.g. Mesh.nodes): torch wants a writable buffer
        arr = arr.copy()
    return t.from_numpy(arr).to(device=device, non_blocking=False)


def is_tensor(a) -> bool:
    try:
        import torch as _t
    except Exception:  # pragma: no cover
        return False
    return isinstance(a, _t.Tensor)
