"""ctypes binding of libalyab200.so (include/alyab200.h).

There is no fallback: if the shared object is missing or does not load, every
entry point of the package raises.  ``call`` turns a negative status into a
``RuntimeError`` carrying ``ab_last_error()``.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libalyab200.so"

RULE_ID = {"tet1": 0, "tet4": 1, "pyr5": 2, "pri6": 3, "hex8": 4}

vp = C.c_void_p
i32 = C.c_int32
i64 = C.c_int64
f64 = C.c_double


class AbCategory(C.Structure):
    _fields_ = [("rule", i32), ("pad_", i32), ("n_elem", i64), ("conn", vp)]


class AbMesh(C.Structure):
    _fields_ = [("n_nodes", i64), ("coords", vp), ("period", f64 * 3), ("n_cat", i32), ("pad_", i32),
                ("cat", AbCategory * 5)]


class AbPhys(C.Structure):
    _fields_ = [("rho", f64), ("mu", f64), ("c_vreman", f64)]


class AbSell(C.Structure):
    _fields_ = [("n_rows", i64), ("n_slices", i64), ("max_width", i64), ("slice_ptr", vp), ("cols", vp),
                ("vals", vp)]


class AbSell3(C.Structure):
    _fields_ = [("n_rows", i64), ("n_slices", i64), ("slice_ptr", vp), ("cols", vp), ("vx", vp), ("vy", vp),
                ("vz", vp)]


class AbWall(C.Structure):
    _fields_ = [("n_faces", i64), ("face", vp), ("off", vp), ("n_nodes", i64), ("node", vp), ("ptr", vp),
                ("fref", vp), ("ftrac", vp)]


class AbCgLocal(C.Structure):
    _fields_ = [("rows_per_cta", i64), ("n_cta", i32), ("max_ghost", i32), ("cols", vp), ("ghost_ptr", vp),
                ("ghost", vp), ("perm", vp), ("prefetch_depth", i32),
                ("variant", i32), ("packed", vp), ("group", i32), ("force_mode", i32),
                ("nbr_ptr", vp), ("nbr", vp)]


PEER_MAX = 8
u64p = C.c_void_p


class AbPeerHalo(C.Structure):
    _fields_ = ([("rank", i32), ("n_ranks", i32), ("n_if", i32), ("n_cta", i32), ("max_shared", i32), ("n_nbr", i32)]
                + [(n, vp) for n in ("if_node", "if_ptr", "if_rank", "if_slot", "recv", "cnt_in", "state")]
                + [("nbr_rank", i32 * PEER_MAX), ("nbr_ncta", i32 * PEER_MAX), ("nbr_recv", vp * PEER_MAX),
                   ("nbr_cnt", vp * PEER_MAX)])


class AbDdcg2Rank(C.Structure):
    _fields_ = ([("n_rows", i64), ("n_if", i64), ("rank", i32), ("n_ranks", i32), ("n_peers", i32),
                 ("recv_stride", i32)]
                + [(n, vp) for n in ("slice_ptr", "cols", "vals", "dinv", "fixed", "own", "s", "perm", "x", "r", "z",
                                     "p", "q", "tif", "send_ptr", "send_peer", "send_off", "recv_ptr", "recv_rank",
                                     "recv_off", "recv", "cnt_in", "rec", "part", "cnt", "scal")]
                + [("nsig", i32), ("scaled", i32), ("peer_rank", i32 * PEER_MAX), ("peer_nsig", i32 * PEER_MAX),
                   ("peer_recv", vp * PEER_MAX), ("peer_cnt", vp * PEER_MAX), ("peer_rec", vp * PEER_MAX),
                   ("tcols", vp), ("tghost_ptr", vp), ("tghost", vp), ("tile_rows", i32), ("tmax_ghost", i32),
                   ("xp", vp), ("rq", vp * 2), ("single_pass", i32), ("pad_sp_", i32)])


class AbMeshDesc(C.Structure):
    _fields_ = [("n_nodes", i64), ("coords", vp), ("period", f64 * 3), ("n_cat", i32), ("pad_", i32),
                ("cat", AbCategory * 5), ("p_fixed", vp), ("u_fixed", vp), ("u_values", vp), ("n_wall_faces", i64),
                ("wall_face", vp), ("wall_off", vp), ("phys", AbPhys)]


class AbCtxInfo(C.Structure):
    _fields_ = [("n_nodes", i64), ("nnz", i64), ("n_cat", i32), ("ready", i32), ("n_elem", i64 * 5),
                ("n_velocity_bc", i64), ("n_wall_faces", i64)]


P = C.POINTER
_SIGS = {
    "ab_ctx_create": ([i32, vp], C.c_int),
    "ab_ctx_destroy": ([vp], C.c_int),
    "ab_mesh_upload": ([vp, P(AbMeshDesc)], C.c_int),
    "ab_ctx_info": ([vp, P(AbCtxInfo)], C.c_int),
    "ab_state_set": ([vp, vp, vp, vp], C.c_int),
    "ab_state_get": ([vp, vp, vp, vp], C.c_int),
    "ab_step": ([vp, f64, i32, vp], C.c_int),
    "ab_peer_halo_put": ([P(AbPeerHalo), vp, i32, i32, vp], C.c_int),
    "ab_peer_halo_add": ([P(AbPeerHalo), vp, i32, i32, vp], C.c_int),
    "ab_peer_halo_grid": ([i32], C.c_int),
    "ab_ddcg2_init": ([P(AbDdcg2Rank), vp, vp, f64, vp], C.c_int),
    "ab_ddcg2_spmv": ([P(AbDdcg2Rank), vp], C.c_int),
    "ab_ddcg2_iface": ([P(AbDdcg2Rank), vp], C.c_int),
    "ab_ddcg2_update": ([P(AbDdcg2Rank), vp], C.c_int),
    "ab_ddcg2_finish": ([P(AbDdcg2Rank), vp, vp], C.c_int),
    "ab_ddcg2_tile_iter": ([P(AbDdcg2Rank), vp], C.c_int),
    "ab_ddcg2_tile_iface": ([P(AbDdcg2Rank), vp], C.c_int),
    "ab_ddcg2_part_size": ([i64], i64),
    "ab_version": ([], C.c_int),
    "ab_last_error": ([], C.c_char_p),
    "ab_launch_count": ([], i64),
    "ab_set_windows": ([vp, i32, vp, vp, vp, vp, vp, vp, i32], C.c_int),
    "ab_set_window_refs": ([vp, vp], C.c_int),
    "ab_set_window_colours": ([vp, i32, vp, vp, vp], C.c_int),
    "ab_colour_blocks": ([i64, vp, vp, vp, vp, vp, vp, vp], C.c_int),
    "ab_format_partition": ([vp, i64, i64, vp, i64], C.c_int64),
    "ab_filter_width": ([P(AbMesh), i32, vp, vp], C.c_int),
    "ab_set_filter_width": ([vp, i64, vp], C.c_int),
    "ab_parse_partition": ([vp, i64, vp, i64, vp], C.c_int64),
    "ab_mass": ([P(AbMesh), i32, vp, vp, vp, i32, vp], C.c_int),
    "ab_last_pipe_shape": ([vp, vp], C.c_int),
    "ab_momentum_rhs": ([P(AbMesh), P(AbPhys), vp, vp, vp], C.c_int),
    "ab_divergence": ([P(AbMesh), vp, f64, vp, vp], C.c_int),
    "ab_wall_traction": ([P(AbWall), P(AbPhys), vp, vp, vp, vp], C.c_int),
    "ab_gradient": ([P(AbMesh), vp, f64, vp, vp], C.c_int),
    "ab_laplacian_csr": ([P(AbMesh), vp, vp, vp, vp], C.c_int),
    "ab_csr_dirichlet": ([i64, vp, vp, vp, vp, vp], C.c_int),
    "ab_csr_to_sell": ([i64, vp, vp, vp, vp, vp, vp, vp, vp], C.c_int),
    "ab_sell_spmv": ([P(AbSell), vp, vp, vp], C.c_int),
    "ab_cg_init": ([i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp], C.c_int),
    "ab_cg_set_bb": ([vp, vp, vp], C.c_int),
    "ab_sell_symscale": ([P(AbSell), vp, vp], C.c_int),
    "ab_cg_spmv_unit": ([P(AbSell), vp, vp, vp, vp, vp, vp, vp, vp], C.c_int),
    "ab_cg_init_scaled": ([i64, vp, vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp], C.c_int),
    "ab_cg_update_scaled": ([i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp], C.c_int),
    "ab_cg_finish_scaled": ([i64, vp, vp, vp, vp, vp], C.c_int),
    "ab_cg_spmv_tile": ([P(AbSell), P(AbCgLocal), vp, vp, vp, vp, vp, vp, vp, vp], C.c_int),
    "ab_cg_tile_init": ([i64, vp, vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp], C.c_int),
    "ab_cg_tile_iter": ([P(AbSell), P(AbCgLocal), vp, vp, vp, vp, vp, vp, vp, vp], C.c_int),
    "ab_cg_tile_finish": ([i64, vp, vp, vp, vp, i32, vp, vp], C.c_int),
    "ab_cg_init_perm": ([i64, vp, vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp], C.c_int),
    "ab_perm_scatter": ([i64, vp, vp, vp, vp], C.c_int),
    "ab_cg_spmv": ([P(AbSell), vp, vp, vp, vp, i32, vp, vp, vp, vp, vp, vp], C.c_int),
    "ab_cg_dot": ([i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp], C.c_int),
    "ab_cg_update": ([i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp], C.c_int),
    "ab_cg_resident_fits": ([i64, vp, vp], C.c_int),
    "ab_cg_resident_local_fits": ([i64, i32], C.c_int),
    "ab_debug_timeline": ([vp], C.c_int),
    "ab_cg_resident_local": ([P(AbSell), P(AbCgLocal), vp, vp, vp, vp, vp, vp, i32, f64, vp, vp, vp, vp],
                             C.c_int),
    "ab_gradop_csr": ([P(AbMesh), vp, vp, vp, vp, vp, vp], C.c_int),
    "ab_gradop_div": ([P(AbSell3), vp, f64, vp, vp], C.c_int),
    "ab_gradop_grad": ([P(AbSell3), vp, f64, vp, vp], C.c_int),
    "ab_gradop_correct": ([P(AbSell3), vp, f64, vp, vp, vp, vp, vp, vp], C.c_int),
    "ab_cg_dd": ([vp, i32, i32, i32, f64, i64, i32, vp], C.c_int),
    "ab_ipc_get_handle": ([vp, vp, vp], C.c_int),
    "ab_ipc_open_handle": ([vp, vp], C.c_int),
    "ab_ipc_close": ([vp], C.c_int),
    "ab_rk_stage": ([i64, f64, f64, f64, vp, vp, vp, vp, vp, vp, vp], C.c_int),
    "ab_correct": ([i64, f64, vp, vp, vp, vp, vp, vp, vp, vp], C.c_int),
    "ab_apply_velocity_bc": ([i64, vp, vp, vp, vp, vp], C.c_int),
    "ab_reciprocal": ([i64, vp, vp, vp], C.c_int),
    "ab_halo_pack": ([i64, vp, vp, i32, i32, vp, vp], C.c_int),
    "ab_halo_unpack_add": ([i64, vp, vp, i32, i32, vp, vp], C.c_int),
    "ab_segment_sum": ([i64, vp, vp, vp, vp], C.c_int),
    "ab_centroids": ([P(AbMesh), i32, vp, vp], C.c_int),
    "ab_hilbert_keys": ([i64, vp, vp, vp, i32, vp, vp], C.c_int),
    "ab_hilbert_cells": ([i64, vp, i32, vp, vp], C.c_int),
}

EXPORTED = tuple(_SIGS)
_lib = None


def lib():
    """Load (once) and return the CDLL; raises if the library is missing."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_2005_05899_b200.build` "
                               "(there is no CPU fallback)")
        dll = C.CDLL(str(LIB_PATH))
        for name, (args, res) in _SIGS.items():
            fn = getattr(dll, name)
            fn.argtypes = args
            fn.restype = res
        _lib = dll
    return _lib


def call(name: str, *args) -> None:
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        msg = lib().ab_last_error().decode(errors="replace")
        raise RuntimeError(f"{name} failed ({rc}): {msg}")


def launch_count() -> int:
    return int(lib().ab_launch_count())


def ptr(t) -> int | None:
    """Raw device pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_handle(stream=None) -> int:
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream
