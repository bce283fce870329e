"""ctypes binding of libemhd.so (the C ABI in include/emhd.h).

There is no CPU fallback: importing the compute entry points without the
built library, or without a CUDA device, raises immediately.
"""

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# EMHD_LIB: an alternative in-tree build of the same ABI (A/B kernel experiments)
LIB_PATH = os.environ.get("EMHD_LIB") or os.path.join(HERE, "libemhd.so")

c_int, c_ll, c_dbl, c_vp = ctypes.c_int, ctypes.c_longlong, ctypes.c_double, ctypes.c_void_p
P = ctypes.c_void_p          # device pointers travel as integers
PP = ctypes.POINTER(ctypes.c_void_p)
IP = ctypes.POINTER(ctypes.c_int)
DP = ctypes.POINTER(ctypes.c_double)


class Geometry(ctypes.Structure):
    _fields_ = [("nx", c_int), ("ny", c_int), ("nx_global", c_int), ("x_offset", c_int),
                ("hx", c_dbl), ("hy", c_dbl), ("bc_x_lo", c_int), ("bc_x_hi", c_int),
                ("bc_y", c_int)]


class Physics(ctypes.Structure):
    _fields_ = [("mu", c_dbl), ("eta", c_dbl), ("kappa", c_dbl), ("gamma", c_dbl),
                ("b_half", c_int), ("check", c_int)]


class Status(ctypes.Structure):
    _fields_ = [("flags", c_int), ("rhs_evals", c_int), ("first_nonfinite", ctypes.c_ulonglong),
                ("breakdown", c_int), ("fail_iter", c_int), ("rhs_evals_mark", c_int)]


class ArnoldiArgs(ctypes.Structure):
    _fields_ = [("a", P), ("fa", P), ("V", P), ("ldv", c_ll), ("H", P), ("ldh", c_ll),
                ("w0", P), ("w1", P), ("d1", P), ("d2", P), ("nrm", P), ("vn", P), ("scal", P),
                ("brk", P), ("n_top", c_ll), ("len_dot", c_ll), ("len_upd", c_ll), ("p", c_int),
                ("nb", c_int), ("ch", c_dbl), ("bcol", P * 5), ("bidx", c_int * 5),
                ("gen", c_int), ("gate", P), ("evals", P), ("eta", c_dbl), ("reorth", P),
                ("md2", P), ("a_halo", P)]


class StencilPath(ctypes.Structure):
    _fields_ = [("kernel", c_int), ("rows_per_cta", c_int), ("strip", c_int), ("bulk", c_int),
                ("min_rows", c_int), ("tile_rows", c_int), ("raw_rows", c_int)]


STENCIL_AUTO, STENCIL_MARCHING, STENCIL_TILE = 0, 1, 2


class Report(ctypes.Structure):
    _fields_ = [("which", c_int), ("i", c_int), ("j", c_int), ("pad", c_int), ("value", c_dbl)]


ST_RHO, ST_PRESSURE, ST_NONFINITE, ST_BREAKDOWN, ST_DENSE = 1, 2, 4, 8, 16
OP_SUM, OP_MAX, OP_MIN = 0, 2, 3
HostAllreduceFn = ctypes.CFUNCTYPE(c_int, c_vp, DP, c_int, c_int)
HostExchangeFn = ctypes.CFUNCTYPE(c_int, c_vp, DP, DP, c_ll)
BC = {"periodic": 0, "reflect": 1, "zero-gradient": 2, "external": 3}

_SIGS = {
    "emhd_version": (ctypes.c_char_p, []),
    "emhd_error_string": (ctypes.c_char_p, [c_int]),
    "emhd_ctx_create": (c_int, [ctypes.POINTER(c_vp), ctypes.POINTER(Geometry),
                                ctypes.POINTER(Physics), c_int]),
    "emhd_ctx_destroy": (c_int, [c_vp]),
    "emhd_set_stream": (c_int, [c_vp, c_vp]),
    "emhd_num_sms": (c_int, [c_vp]),
    "emhd_status_read": (c_int, [c_vp, ctypes.POINTER(Status)]),
    "emhd_status_reset": (c_int, [c_vp]),
    "emhd_status_scrub": (c_int, [c_vp, c_int]),
    "emhd_evals_mark": (c_int, [c_vp]),
    "emhd_status_clear_errors": (c_int, [c_vp]),
    "emhd_set_stencil_path": (c_int, [c_vp, ctypes.POINTER(StencilPath)]),
    "emhd_get_stencil_path": (c_int, [c_vp, ctypes.POINTER(StencilPath)]),
    "emhd_set_fused_orth": (c_int, [c_vp, c_int]),
    "emhd_last_stencil": (c_int, [c_vp, ctypes.POINTER(StencilPath)]),
    "emhd_rhs": (c_int, [c_vp, P, P, P]),
    "emhd_jv": (c_int, [c_vp, P, P, P, P, P, P, P]),
    "emhd_jv_aug": (c_int, [c_vp, P, P, P, P, P, P, P, c_int, c_dbl, c_int, PP, IP, P]),
    "emhd_jv_normalized": (c_int, [c_vp, P, P, P, P, P, P, P, c_int, c_dbl, c_int, PP, IP, P]),
    "emhd_multidot": (c_int, [c_vp, P, P, c_ll, c_int, c_ll, c_int, P]),
    "emhd_update": (c_int, [c_vp, P, P, c_ll, c_int, P, c_ll, c_ll, c_ll, c_int, P]),
    "emhd_norms": (c_int, [c_vp, P, c_ll, c_ll, P]),
    "emhd_update_finish": (c_int, [c_vp, P, P, c_ll, c_int, P, c_ll, c_ll, c_ll, P, P, P, c_int, P,
                                   c_ll, P, P]),
    "emhd_arnoldi_finish": (c_int, [c_vp, P, P, P, P, c_int, P, c_ll, P, P]),
    "emhd_set_epoch": (c_int, [c_vp, c_int]),
    "emhd_div_scalar": (c_int, [c_vp, P, P, c_int, P, P, c_ll]),
    "emhd_phi_small": (c_int, [c_vp, P, c_ll, c_int, c_int, c_int, P, P, P, P, P, P]),
    "emhd_expm": (c_int, [c_vp, P, c_int, P, P]),
    "emhd_phi_small_h": (c_int, [c_vp, P, c_ll, c_int, c_int, c_int, DP, P, P, P, P]),
    "emhd_arnoldi_iter": (c_int, [c_vp, c_vp, c_int]),
    "emhd_arnoldi_run": (c_int, [c_vp, c_vp, c_int, c_int]),
    "emhd_arnoldi_lookahead": (c_int, [c_vp, c_vp, c_int, c_int]),
    "emhd_arnoldi_cancel": (c_int, [c_vp, c_int, c_int]),
    "emhd_evals_discount": (c_int, [c_vp, P, c_int]),
    "emhd_phi_small_batch": (c_int, [c_vp, P, c_ll, IP, c_int, c_int, DP, P, P, P, c_ll, P]),
    "emhd_readback": (c_int, [c_vp, P, c_int, P, c_int, P, ctypes.POINTER(Status)]),
    "emhd_combine": (c_int, [c_vp, P, c_ll, c_int, P, c_int, PP, DP, PP, c_ll]),
    "emhd_lincomb": (c_int, [c_vp, c_int, PP, DP, IP, c_dbl, c_int, P, c_ll, c_ll, P]),
    "emhd_wrms": (c_int, [c_vp, P, P, c_dbl, c_ll, P]),
    "emhd_pack_edges": (c_int, [c_vp, P, P]),
    "emhd_slot_norms": (c_int, [c_vp, P, c_int, c_int, P]),
    "emhd_reorth_decide": (c_int, [c_vp, P, P, c_int, P, c_int, P, c_ll, P, P, c_dbl, P]),
    "emhd_skip_next": (c_int, [c_vp, P]),
    "emhd_l2_window": (c_int, [c_vp, P, c_ll]),
    "emhd_profile": (c_int, [c_vp, c_int]),
    "emhd_profile_read": (c_int, [c_vp, c_int, IP, DP, DP]),
    "emhd_push_edges": (c_int, [c_vp, P, P, P, P]),
    "emhd_update_push": (c_int, [c_vp, P, P, c_ll, c_int, P, c_ll, c_ll, c_ll, P, P, P]),
    "emhd_unslot_norms": (c_int, [c_vp, P, c_int, P]),
    "emhd_div_b": (c_int, [c_vp, P, P, P, P]),
    "emhd_current_j": (c_int, [c_vp, P, P, P]),
    "emhd_admissibility_report": (c_int, [c_vp, c_int, P, P, P, P, P, ctypes.POINTER(Report)]),
    "emhd_cells_pack": (c_int, [c_vp, P, c_ll, P]),
    "emhd_cells_unpack": (c_int, [c_vp, P, c_ll, P]),
    "emhd_max_signal_speed": (c_int, [c_vp, P, P]),
    "emhd_field_sqdiff": (c_int, [c_vp, P, P, P]),
    "emhd_lincomb_onto": (c_int, [c_vp, P, c_int, PP, DP, IP, c_dbl, c_int, P, c_ll]),
    "emhd_nccl_unique_id": (c_int, [ctypes.c_char_p]),
    "emhd_comm_init_nccl": (c_int, [c_vp, c_int, c_int, c_int, c_int, ctypes.c_char_p, ctypes.c_char_p]),
    "emhd_comm_init_host": (c_int, [c_vp, c_int, c_int, c_int, c_int, HostAllreduceFn, HostExchangeFn,
                                    c_vp]),
    "emhd_allreduce": (c_int, [c_vp, P, c_int, c_int]),
    "emhd_halo_exchange": (c_int, [c_vp, P, P]),
    "emhd_set_dense_cluster": (c_int, [c_int]),
    "emhd_set_dense_gj_blocked": (c_int, [c_int]),
}

_lib = None


class NativeError(RuntimeError):
    pass


def lib():
    """The loaded libemhd.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1604_02614_b200.build` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return list(_SIGS)


def check(rc, what=""):
    if rc != 0:
        msg = lib().emhd_error_string(rc).decode()
        raise NativeError(f"libemhd {what} failed: {msg} (code {rc})")


def ptr_array(ptrs):
    arr = (ctypes.c_void_p * max(1, len(ptrs)))()
    for k, p in enumerate(ptrs):
        arr[k] = p
    return arr


def int_array(vals):
    arr = (ctypes.c_int * max(1, len(vals)))()
    for k, v in enumerate(vals):
        arr[k] = int(v)
    return arr


def dbl_array(vals):
    arr = (ctypes.c_double * max(1, len(vals)))()
    for k, v in enumerate(vals):
        arr[k] = float(v)
    return arr
