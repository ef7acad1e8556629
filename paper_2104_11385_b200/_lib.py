"""ctypes binding of libLBX (include/lbx.h).

There is deliberately no fallback: if the shared library is missing or was
built without a symbol, importing the package fails with an error that says
how to build it.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import ConfigError  # noqa: F401  (re-exported for callers)

LIB_PATH = Path(__file__).resolve().parent / "libLBX.so"
if os.environ.get("LBX_VARIANT"):   # tuning experiments: an in-tree build variant libLBX.<v>.so
    LIB_PATH = LIB_PATH.with_name(f"libLBX.{os.environ['LBX_VARIANT']}.so")

LBX_OK, LBX_EINVAL, LBX_ECUDA, LBX_EOOM, LBX_ERANGE = 0, 1, 2, 3, 4
LBX_STEP_CLOCK = 1

i32, i64, u32, u64, f64 = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_double
vp = C.c_void_p
P = C.POINTER


class StepArgs(C.Structure):
    """lbx_step_args (include/lbx.h)."""
    _fields_ = [("z", vp), ("x", vp), ("vz", vp), ("vx", vp),
                ("extent_z", f64), ("extent_x", f64), ("box_size", f64),
                ("nbz", i32), ("nbx", i32),
                ("w_particle", f64), ("w_cell", f64), ("cells_per_box", f64),
                ("flags", u32),
                ("counts_out", vp), ("cost_out", vp), ("clk_out", vp),
                ("n_out", vp), ("err_out", vp)]


class SimConfig(C.Structure):
    """lbx_sim_config (include/lbx.h)."""
    _fields_ = [("extent_z", i32), ("extent_x", i32), ("box_size", i32), ("n_ranks", i32),
                ("total_steps", i64), ("kick_step", i64),
                ("strategy", i32), ("interval", i64), ("improvement_threshold", f64),
                ("threshold_relative", i32), ("cap_factor", f64), ("static_step", i64),
                ("cost_kind", i32), ("w_particle", f64), ("w_cell", f64),
                ("noise_amplitude", f64), ("noise_seed", u64), ("overhead_factor", f64),
                ("work_wp", f64), ("work_wc", f64),
                ("comm_per_face", f64), ("gather", f64),
                ("redistribute_per_particle", f64), ("redistribute_latency", f64),
                ("capacity_particles", i64), ("physics", i32), ("pic_dt", f64),
                ("pic_q_over_m", f64), ("pic_q_times_w", f64), ("extent_y", i32),
                ("migration_ratio", f64), ("clock_mode", i32)]


class SimOutputs(C.Structure):
    """lbx_sim_outputs (include/lbx.h)."""
    _fields_ = [("eff_before", vp), ("eff_after", vp), ("adopted", vp), ("attempted", vp),
                ("compute_max", vp), ("comm_max", vp), ("gather", vp),
                ("redistribute", vp), ("walltime", vp), ("max_rank_particles", vp),
                ("oom", vp), ("n_alive", vp), ("cost_trace", vp), ("count_trace", vp),
                ("clock_trace", vp), ("owner", vp), ("adopt_steps", vp),
                ("adopt_owners", vp), ("kernel_ms", vp), ("n_adoptions", i64), ("n_attempts", i64),
                ("completed_steps", i64)]


# name -> (restype, argtypes); every symbol include/lbx.h declares.
SIGNATURES = {
    "lbx_last_error": (C.c_char_p, []),
    "lbx_version": (C.c_char_p, []),
    "lbx_ctx_create": (i32, [P(vp), i32, i64]),
    "lbx_ctx_destroy": (i32, [vp]),
    "lbx_ctx_reserve": (i32, [vp, i64]),
    "lbx_ctx_set_count": (i32, [vp, i64, vp]),
    "lbx_ctx_get_count": (i32, [vp, P(i64), vp]),
    "lbx_ctx_set_grid": (i32, [vp, i32]),
    "lbx_ctx_enable_timing": (i32, [vp, i32]),
    "lbx_ctx_last_kernel_ms": (i32, [vp, P(C.c_float)]),
    "lbx_advance_particles": (i32, [vp, vp, vp, i64, f64, f64, vp, vp, vp, vp]),
    "lbx_bin_particles": (i32, [vp, i64, f64, i32, i32, vp, vp, vp]),
    "lbx_push_step": (i32, [vp, P(StepArgs), vp]),
    "lbx_heuristic_cost": (i32, [vp, vp, i64, f64, f64, vp, vp]),
    "lbx_rank_loads": (i32, [vp, vp, i64, i32, vp]),
    "lbx_efficiency": (i32, [vp, vp, i64, i32, P(f64), P(i32)]),
    "lbx_knapsack": (i32, [vp, i64, i32, f64, vp]),
    "lbx_sfc": (i32, [vp, vp, i64, i32, vp]),
    "lbx_morton_order": (i32, [i32, i32, vp]),
    "lbx_morton_order_3d": (i32, [i32, i32, i32, vp]),
    "lbx_slab_mapping": (i32, [i64, i32, vp]),
    "lbx_pairwise_sum": (f64, [vp, i64]),
    "lbx_measured_cost": (i32, [vp, i64, f64, u64, u64, vp]),
    "lbx_sim_create": (i32, [P(vp), vp, P(SimConfig)]),
    "lbx_sim_destroy": (i32, [vp]),
    "lbx_sim_set_particles": (i32, [vp, vp, vp, vp, vp, vp, vp, i64, vp]),
    "lbx_sim_run": (i32, [vp, i64, i64, P(SimOutputs), vp]),
    "lbx_sim_particles": (i32, [vp, P(i64), vp]),
    "lbx_sim_graph_cycles": (i32, [vp, P(i64)]),
    "lbx_sim_resident_runs": (i32, [vp, P(i64)]),
}


class ExchangeArgs(C.Structure):
    """lbx_exchange_args (include/lbx.h)."""
    _fields_ = [("owner", vp), ("rank", i32), ("world", i32), ("stage", vp),
                ("stage_dest", vp), ("stage_cap", i64), ("send_counts", vp),
                ("kick_vz", vp), ("kick_vx", vp), ("removed_list", vp),
                ("removed_cap", i64), ("peer_recv", vp), ("peer_cursor", vp),
                ("peer_recv_cap", i64)]


SIGNATURES.update({
    "lbx_lb_create": (i32, [P(vp), P(SimConfig), vp]),
    "lbx_lb_destroy": (i32, [vp]),
    "lbx_lb_step": (i32, [vp, i64, vp, vp, i64, P(SimOutputs), P(i32), P(i32)]),
    "lbx_lb_owner": (i32, [vp, vp]),
    "lbx_push_step_exchange": (i32, [vp, P(StepArgs), P(ExchangeArgs), vp]),
    "lbx_partition": (i32, [vp, vp, vp, vp, vp, f64, f64, f64, i32, i32, P(ExchangeArgs),
                            vp, vp]),
    "lbx_group_by_dest": (i32, [vp, vp, i64, i32, vp, vp, vp]),
    "lbx_unpack": (i32, [vp, i64, i64, vp, vp, vp, vp, vp, vp, vp]),
    "lbx_fill_holes": (i32, [vp, vp, vp, vp, vp, vp, vp, vp, i64, i64, vp]),
    "lbx_advance_bin_host": (i32, [vp, vp, vp, i64, f64, f64, f64, i32, i32, f64, f64, vp, vp,
                                   vp, vp, P(i64)]),
})
RECORD_DOUBLES = 6
LBX_PIC_NO_FIELD_SOLVE = 2
LBX_PIC_RESYNC = 4
LBX_PIC_DEFER_CURRENT = 8
LBX_PIC_QUAD = 16
LBX_PIC_STABLE_ORDER = 64
LBX_PIC_DIRECT = 32
LBX_PIC_TILED = 128
LBX_PIC_FAST = 256


class PicArgs(C.Structure):
    """lbx_pic_args (include/lbx.h)."""
    _fields_ = [("z", vp), ("x", vp), ("uz", vp), ("ux", vp), ("uy", vp),
                ("fields", vp * 6), ("current", vp * 3), ("nz", i32), ("nx", i32),
                ("box_size", i32), ("q_over_m", f64), ("q_times_w", f64), ("dt", f64),
                ("w_particle", f64), ("w_cell", f64), ("flags", u32),
                ("counts_out", vp), ("cost_out", vp), ("clk_out", vp), ("n_out", vp),
                ("err_out", vp), ("out", vp * 5), ("shape_order", i32)]


SIGNATURES["lbx_pic_step"] = (i32, [vp, P(PicArgs), vp])
SIGNATURES["lbx_lb_set_migration_ratio"] = (i32, [vp, f64])
SIGNATURES["lbx_pic_sort"] = (i32, [vp, P(PicArgs), vp])
SIGNATURES["lbx_peer_alloc"] = (i32, [i64, P(vp), vp])
SIGNATURES["lbx_ctx_set_upper"] = (i32, [vp, i64])
SIGNATURES["lbx_fill_holes_dev"] = (i32, [vp, vp, vp, vp, vp, vp, vp, vp, i64, f64, f64, vp])
SIGNATURES["lbx_unpack_peer_dev"] = (i32, [vp, vp, vp, i64, vp, vp, vp, vp, vp, vp, vp])
SIGNATURES["lbx_peer_open"] = (i32, [vp, P(vp)])
SIGNATURES["lbx_peer_close"] = (i32, [vp])
SIGNATURES["lbx_peer_free"] = (i32, [vp])
SIGNATURES["lbx_peer_can_access"] = (i32, [i32, i32, P(i32)])
SIGNATURES["lbx_pic_finish"] = (i32, [vp, P(PicArgs), vp])
SIGNATURES["lbx_pic_current_view"] = (i32, [vp, P(vp), P(i64), P(vp)])
SIGNATURES["lbx_pic_esk_current_view"] = (i32, [vp, P(vp), P(i64), P(i32)])
SIGNATURES["lbx_sim_set_fields"] = (i32, [vp, vp, vp, vp])


class Step3DArgs(C.Structure):
    """lbx_step3d_args (include/lbx.h)."""
    _fields_ = [("z", vp), ("y", vp), ("x", vp), ("vz", vp), ("vy", vp), ("vx", vp),
                ("extent_z", i32), ("extent_y", i32), ("extent_x", i32), ("box_size", i32),
                ("w_particle", f64), ("w_cell", f64), ("flags", u32), ("counts_out", vp),
                ("cost_out", vp), ("clk_out", vp), ("n_out", vp), ("err_out", vp),
                ("removed_list", vp), ("removed_cap", i64)]


SIGNATURES["lbx_push_step_3d"] = (i32, [vp, P(Step3DArgs), vp])
SIGNATURES["lbx_push_step_3d_exchange"] = (i32, [vp, P(Step3DArgs), P(ExchangeArgs), vp])
SIGNATURES["lbx_partition_3d"] = (i32, [vp, vp, vp, vp, vp, vp, vp, i32, i32, i32, i32,
                                        P(ExchangeArgs), vp, vp])


class LBXError(RuntimeError):
    pass


def _load():
    if not LIB_PATH.exists():
        raise ImportError(
            f"libLBX not built ({LIB_PATH} missing). Run "
            "`python -c 'import __graft_entry__ as g; g.build()'` from the repo "
            "root (needs nvcc with sm_100a). There is no CPU fallback.")
    lib = C.CDLL(str(LIB_PATH))
    missing = []
    for name, (res, args) in SIGNATURES.items():
        try:
            fn = getattr(lib, name)
        except AttributeError:
            missing.append(name)
            continue
        fn.restype = res
        fn.argtypes = args
    if missing:
        raise ImportError(f"libLBX at {LIB_PATH} lacks symbols {missing}; rebuild it")
    return lib


lib = _load()


def check(rc: int) -> None:
    """Map a libLBX return code onto the reference's exception classes."""
    if rc == LBX_OK:
        return
    msg = lib.lbx_last_error().decode()
    if rc in (LBX_EINVAL, LBX_ERANGE):
        raise ValueError(msg)
    if rc == LBX_EOOM:
        raise MemoryError(msg)
    raise LBXError(msg)


def ptr(a) -> int:
    """Address of a numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data
