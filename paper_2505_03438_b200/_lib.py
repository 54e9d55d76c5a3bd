"""ctypes binding of libmdg (include/mdg.h).

The library is built in-tree (``paper_2505_03438_b200/_build/libmdg.so``) by
``__graft_entry__.build()`` / ``make -C paper_2505_03438_b200/csrc``.  There
is no fallback: if the library is missing or cannot load, every GPU entry
point raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MDG_LIB_PATH") or os.path.join(_HERE, "_build", "libmdg.so")

MDG_OK, MDG_EINVAL, MDG_ECUDA, MDG_ESTATE = 0, 1, 2, 3
LC, VL, VCL = 0, 1, 2
C01, C08, C18, SLI, LIST_ITER, CLUSTER_ITER = 0, 1, 2, 3, 4, 5
AOS, SOA = 0, 1

# every symbol include/mdg.h declares (tests check the export list)
EXPORTS = (
    "mdg_version", "mdg_launch_count", "mdg_last_error", "mdg_create", "mdg_destroy", "mdg_set_stream",
    "mdg_set_system", "mdg_bind", "mdg_rebuild", "mdg_refresh", "mdg_compute",
    "mdg_eval_count", "mdg_potential_energy", "mdg_drift_wrap", "mdg_finish_kick", "mdg_sd_step", "mdg_blowup",
    "mdg_profile", "mdg_profile_read", "mdg_synchronize", "mdg_h2d", "mdg_d2h", "mdg_geometry", "mdg_stencil", "mdg_get_grid",
    "mdg_get_verlet", "mdg_geometry_for", "mdg_stencil_for", "mdg_host_drift_wrap",
    "mdg_host_finish_kick", "mdg_measure_fp64_peak", "mdg_temperature", "mdg_thermostat",
    "mdg_live_stats", "mdg_compute_kick", "mdg_step_graph", "mdg_host_step", "mdg_host_step_ex",
    "mdg_host_run", "mdg_host_kick_drift_range", "mdg_kick_drift", "mdg_lc_pairs", "mdg_timings",
    "mdg_host_drift_wrap_range_ex", "mdg_d2h_async", "mdg_host_drift_wrap_range", "mdg_host_finish_kick_range",
    "mdg_set_prune", "mdg_prune_count", "mdg_rebuild_checked", "mdg_owned_order",
    "mdg_ghost_pack", "mdg_ghost_unpack", "mdg_gather_rows", "mdg_set_force_rows",
    "mdg_set_iteration", "mdg_blowup_iteration", "mdg_run", "mdg_permutation",
)
FLAG_BLOWUP, FLAG_THERMO_ZERO = 1, 2


class MdgConfig(ctypes.Structure):
    _fields_ = [("container", ctypes.c_int), ("traversal", ctypes.c_int),
                ("newton3", ctypes.c_int), ("layout", ctypes.c_int), ("csf", ctypes.c_double),
                ("precision", ctypes.c_int)]


class MdgError(RuntimeError):
    pass


_lib = None


def _declare(L):
    P, I, I64, D, SZ = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_size_t
    CFG = ctypes.POINTER(MdgConfig)
    sig = {
        "mdg_version": (ctypes.c_char_p, []),
        "mdg_launch_count": (ctypes.c_uint64, []),
        "mdg_last_error": (ctypes.c_char_p, []),
        "mdg_create": (I, [I, P, ctypes.POINTER(P)]),
        "mdg_destroy": (I, [P]),
        "mdg_set_stream": (I, [P, P]),
        "mdg_set_system": (I, [P, P, P, D, D, I, P, P, P]),
        "mdg_bind": (I, [P, I64, I, P, P, P, P, P]),
        "mdg_rebuild": (I, [P, CFG]),
        "mdg_refresh": (I, [P, CFG]),
        "mdg_compute": (I, [P, CFG]),
        "mdg_eval_count": (I, [P, ctypes.POINTER(I64)]),
        "mdg_potential_energy": (I, [P, I, ctypes.POINTER(D)]),
        "mdg_drift_wrap": (I, [P, D]),
        "mdg_finish_kick": (I, [P, D, I, D]),
        "mdg_sd_step": (I, [P, D, D]),
        "mdg_blowup": (I, [P, ctypes.POINTER(I), I]),
        "mdg_profile": (I, [P, I]),
        "mdg_profile_read": (I, [P, ctypes.POINTER(D), ctypes.POINTER(I64)]),
        "mdg_synchronize": (I, [P]),
        "mdg_h2d": (I, [P, P, P, SZ]),
        "mdg_d2h": (I, [P, P, P, SZ]),
        "mdg_geometry": (I, [P, D, P, P, P, P, P]),
        "mdg_stencil": (I, [P, D, I, I, ctypes.POINTER(I), P]),
        "mdg_get_grid": (I, [P, D, ctypes.POINTER(I64), ctypes.POINTER(I64), P, P, P]),
        "mdg_get_verlet": (I, [P, ctypes.POINTER(I64), P, P]),
        "mdg_geometry_for": (I, [P, P, D, D, P, P, P, P, P]),
        "mdg_stencil_for": (I, [P, P, D, D, I, I, ctypes.POINTER(I), P]),
        "mdg_host_drift_wrap": (I, [I64, I, P, P, P, P, P, P, P, P, D, ctypes.POINTER(I)]),
        "mdg_host_finish_kick": (I, [I64, I, P, P, P, P, P, D, I, D]),
        "mdg_measure_fp64_peak": (I, [P, ctypes.POINTER(D), ctypes.POINTER(D)]),
        "mdg_temperature": (I, [P, ctypes.POINTER(D)]),
        "mdg_thermostat": (I, [P, D, D]),
        "mdg_live_stats": (I, [P, P]),
        "mdg_d2h_async": (I, [P, P, P, SZ]),
        "mdg_compute_kick": (I, [P, CFG, D, I, D]),
        "mdg_step_graph": (I, [P, CFG, D, I, D]),
        "mdg_host_step": (I, [P, CFG, P, P, P, P, P, P, D, I, D, I, I, ctypes.POINTER(I)]),
        "mdg_host_step_ex": (I, [P, CFG, P, P, P, P, P, P, D, I, D, I, I, I, ctypes.POINTER(I)]),
        "mdg_kick_drift": (I, [P, D, I, D, I]),
        "mdg_lc_pairs": (I, [P, D, I64, P, ctypes.POINTER(I64)]),
        "mdg_timings": (I, [P, I, ctypes.POINTER(I64), ctypes.POINTER(I64)]),
        "mdg_set_prune": (I, [P, D]),
        "mdg_rebuild_checked": (I, [P, CFG, ctypes.POINTER(I)]),
        "mdg_owned_order": (I, [P, CFG, P]),
        "mdg_prune_count": (I, [P, ctypes.POINTER(I64)]),
        "mdg_ghost_pack": (I, [P, P, I64, I64, I, D, D, P]),
        "mdg_ghost_unpack": (I, [P, P, I64, I64]),
        "mdg_gather_rows": (I, [P, P, I64, I, P, P, P, P]),
        "mdg_set_force_rows": (I, [P, I64]),
        "mdg_set_iteration": (I, [P, I64]),
        "mdg_blowup_iteration": (I, [P, ctypes.POINTER(I64)]),
        "mdg_permutation": (I, [P, I, I64, P, P, P]),
        "mdg_run": (I, [P, CFG, I64, D, I, D, I, I64, I, ctypes.POINTER(I), ctypes.POINTER(I),
                        ctypes.POINTER(I), ctypes.POINTER(I64), ctypes.POINTER(I)]),
        "mdg_host_run": (I, [P, CFG, P, P, P, P, P, P, D, I, D, I, I, I, I, I, ctypes.POINTER(I),
                             ctypes.POINTER(I)]),
        "mdg_host_kick_drift_range": (I, [I64, I64, I64, I, P, P, P, P, P, P, P, P, D, I, D,
                                          ctypes.POINTER(I)]),
        "mdg_host_drift_wrap_range_ex": (I, [I64, I64, I64, I, P, P, P, P, P, P, P, P, D, I, ctypes.POINTER(I)]),
        "mdg_host_drift_wrap_range": (I, [I64, I64, I64, I, P, P, P, P, P, P, P, P, D, ctypes.POINTER(I)]),
        "mdg_host_finish_kick_range": (I, [I64, I64, I64, I, P, P, P, P, P, D, I, D]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args


def lib():
    """The loaded libmdg; raises RuntimeError when it is not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"libmdg is not built ({LIB_PATH}); run __graft_entry__.build() or "
                "make -C paper_2505_03438_b200/csrc")
        L = ctypes.CDLL(LIB_PATH)
        _declare(L)
        _lib = L
    return _lib


def check(status, what=""):
    """Map an ABI status to the reference's exception types."""
    if status == MDG_OK:
        return
    msg = lib().mdg_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if status == MDG_EINVAL:
        raise ValueError(text)
    raise MdgError(text)


def config_struct(config) -> MdgConfig:
    """Any object with the Configuration fields (configuration.py:20-27)."""
    container = {"LC": LC, "VL": VL, "VCL": VCL}[config.container]
    traversal = {"C01": C01, "C08": C08, "C18": C18, "SLI": SLI,
                 "List_Iter": LIST_ITER, "ClusterIter": CLUSTER_ITER}[config.traversal]
    layout = {"AoS": AOS, "SoA": SOA}[config.layout]
    precision = 1 if getattr(config, "precision", "fp64") == "fp32" else 0
    return MdgConfig(container, traversal, int(bool(config.newton3)), layout,
                     float(config.cell_size_factor), precision)
