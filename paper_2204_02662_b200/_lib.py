"""Loader for libpathgcn_b200.so (the sm_100a CUDA path behind the C ABI in
include/pathgcn_b200.h). Builds it in-tree with nvcc when missing or stale;
fails loudly otherwise — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import glob
import os
import shutil
import subprocess
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SO = os.path.join(PKG, "libpathgcn_b200.so")
HEADER = os.path.join(ROOT, "include", "pathgcn_b200.h")

_lock = threading.Lock()
_lib = None


def _sources():
    return glob.glob(os.path.join(PKG, "csrc", "*")) + [HEADER, os.path.join(PKG, "Makefile")]


def stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(s) > t for s in _sources())


def build(force: bool = False, jobs: int = 4) -> str:
    """Compile the CUDA extension for sm_100a (nvcc, in-tree)."""
    if force or stale():
        if shutil.which("nvcc") is None and not os.path.exists("/usr/local/cuda/bin/nvcc"):
            raise RuntimeError("nvcc not found: cannot build libpathgcn_b200.so")
        env = dict(os.environ)
        env["PATH"] = env.get("PATH", "") + ":/usr/local/cuda/bin"
        subprocess.run(["make", "-s", "-C", PKG, f"-j{jobs}"], check=True, env=env)
    return SO


def load() -> C.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            if stale():
                build()
            _lib = C.CDLL(SO)
            _declare(_lib)
        return _lib


u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)
vp = C.c_void_p
H = C.c_void_p  # opaque handles
u32, u64, i32, i64, f64 = C.c_uint32, C.c_uint64, C.c_int, C.c_int64, C.c_double

class PgMat(C.Structure):
    """pg_mat: a device fp32 matrix (rows x cols, row pitch ld floats)."""
    _fields_ = [("data", C.c_void_p), ("rows", C.c_uint64), ("cols", C.c_uint64), ("ld", C.c_uint64)]


matp = C.POINTER(PgMat)

# every symbol of include/pathgcn_b200.h with its ctypes signature
SIGNATURES = {
    "pg_last_error": [C.c_char_p, C.c_size_t],
    "pg_last_error_kind": [u64p],
    "pg_version": [],
    "pg_device_count": [C.POINTER(C.c_int)],
    "pg_set_heavy_min_degree": [u64],
    "pg_set_tuning": [C.c_char_p, i64],
    "pg_gen_rmat": [u32, u64, f64, f64, f64, f64, u64, u32p, u32p],
    "pg_training_set_size": [u32, f64, u64p],
    "pg_sample_training_set": [u32, f64, u64, u32p],
    "pg_edge_list_load": [C.c_char_p, C.POINTER(H)],
    "pg_edge_list_info": [H, u64p, u64p],
    "pg_edge_list_export": [H, u32p],
    "pg_edge_list_destroy": [H],
    "pg_edge_list_write": [C.c_char_p, u32p, u64],
    "pg_graph_load_file": [i32, C.c_char_p, i32, C.POINTER(H)],
    "pg_training_set_load": [C.c_char_p, u32, u32p, u64, u64p],
    "pg_training_set_write": [C.c_char_p, u32p, u64],
    "pg_graph_build": [i32, i64, u32p, u64, i32, C.POINTER(H)],
    "pg_graph_create": [i32, u32, u64p, u32p, f64p, i32, C.POINTER(H)],
    "pg_graph_assign_weights": [H, i32],
    "pg_graph_info": [H, u32p, u64p, u32p, u64p],
    "pg_graph_export": [H, u64p, u32p, f64p],
    "pg_graph_destroy": [H],
    "pg_path_fingerprint": [H, u32p, u64, u64, u64p],
    "pg_frontiers_compute": [H, u32p, u64, u64, C.POINTER(H)],
    "pg_frontiers_size": [H, u64, u64p],
    "pg_frontiers_export": [H, u64, u32p],
    "pg_frontiers_destroy": [H],
    "pg_path_extract": [H, H, u64, C.POINTER(H)],
    "pg_path_info": [H, u64p, u32p, u32p, u64p, u32p, u32p],
    "pg_path_export": [H, u32p, u32p, u32p, u64p, u32p, f64p],
    "pg_path_set_fingerprint": [H, u64],
    "pg_path_get_fingerprint": [H, u64p],
    "pg_path_destroy": [H],
    "pg_gs_regression": [H, f64p, u32p],
    "pg_gs_regression_stats": [u32, u64, f64, f64p, u32p],
    "pg_gs_default_candidates": [u32, u32p, u64p],
    "pg_gs_oracle_cost": [H, u64, i32, f64, u32p, u64, u32p, f64p, u64p],
    "pg_grouping_cost": [H, u64, i32, f64, f64p],
    "pg_gs_oracle_measured": [H, u64, i32, u64, u32p, u64, u32p, f64p, u64p],
    "pg_group": [H, u32, C.POINTER(H)],
    "pg_group_graph": [H, u32, C.POINTER(H)],
    "pg_groups_info": [H, u32p, u64p, u32p],
    "pg_groups_export": [H, u32p, u64p, u64p, u64p],
    "pg_groups_destroy": [H],
    "pg_aggregate_pull": [H, vp, u64, u64, vp, u64, u64, C.c_uint, vp],
    "pg_backward_aggregate": [H, vp, u64, u64, vp, u64, u64, C.c_uint, vp],
    "pg_backward_aggregate_rows": [H, u32, u32, vp, u64, u64, vp, u64, u64, C.c_uint, vp],
    "pg_aggregate_pull_host": [H, f32p, u64, u64, f32p, C.c_uint, u64p],
    "pg_backward_aggregate_host": [H, f32p, u64, u64, f32p, C.c_uint, u64p],
    "pg_stage_counters": [H, u64, C.c_uint, u64p],
    "pg_path_shard_bounds": [H, u32, u32p],
    "pg_groups_remap_sources": [H, u32p, u64, u64],
    "pg_groups_set_segments": [H, u64p, u32],
    "pg_backward_aggregate_segment": [H, u32, u32, u32, vp, u64, u64, vp, u64, u64, C.c_uint, vp],
    "pg_gemm_a_bt": [vp, u64, vp, u64, vp, u64, u64, u64, u64, vp],
    "pg_aggregate_pull_f64": [H, vp, u64, u64, vp, u64, u64, C.c_uint, vp],
    "pg_backward_aggregate_f64": [H, vp, u64, u64, vp, u64, u64, C.c_uint, vp],
    "pg_aggregate_pull_host_f64": [H, f64p, u64, u64, f64p, C.c_uint, u64p],
    "pg_backward_aggregate_host_f64": [H, f64p, u64, u64, f64p, C.c_uint, u64p],
    "pg_comm_unique_id": [vp],
    "pg_comm_init_rank": [C.c_int, vp, C.c_int, C.c_int, C.POINTER(H)],
    "pg_comm_info": [H, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)],
    "pg_comm_destroy": [H],
    "pg_comm_allgather_rows": [H, vp, u64, u32p, vp],
    "pg_backward_aggregate_sharded": [H, H, u32p, u32p, vp, u64, u64, vp, u64, u64, C.c_uint, vp],
    "pg_gemm_a_bt_ex": [vp, u64, vp, u64, vp, u64, u64, u64, u64, C.c_uint, vp],
    "pg_relu_backward": [vp, u64, vp, u64, vp, u64, u64, u64, vp],
    "pg_gather_rows": [vp, u64, vp, u64, vp, u64, u64, vp],
    "pg_path_device_arrays": [H, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)],
    "pg_device_alloc": [i32, u64, C.POINTER(vp)],
    "pg_device_free": [i32, vp],
    "pg_memcpy_h2d": [i32, vp, vp, u64],
    "pg_memcpy_d2h": [i32, vp, vp, u64],
    "pg_memset_zero": [i32, vp, u64],
    "pg_device_synchronize": [i32],
    "pg_launch_count": [],
    "pg_mat_upload": [i32, PgMat, f32p],
    "pg_mat_download": [i32, f32p, PgMat],
    "pg_gemm": [PgMat, PgMat, i32, PgMat, vp],
    "pg_gemm_at_b": [PgMat, vp, PgMat, PgMat, vp],
    "pg_gemm_at_b_ex": [PgMat, vp, PgMat, PgMat, C.c_uint, vp],
    "pg_relu": [PgMat, PgMat, vp],
    "pg_row_softmax": [PgMat, PgMat, vp],
    "pg_top_grad_from_probs": [PgMat, PgMat, vp, u64, PgMat, vp],
    "pg_aggregate_pull_filtered": [H, H, u64, u64, vp, u64, u64, vp, u64, u64, C.c_uint, u64p, vp],
    "pg_forward": [H, PgMat, matp, u64, matp, matp, matp, vp],
    "pg_backward_epp": [C.POINTER(H), H, u64, matp, matp, PgMat, matp, u64, i32, matp, matp, u64p, vp],
    "pg_backward_all_active": [H, u64, matp, matp, PgMat, matp, matp, matp, u64p, vp],
    "pg_backward_ifelse": [H, H, u64, matp, matp, PgMat, matp, matp, matp, u64p, vp],
}


def header_symbols():
    """Function names declared in include/pathgcn_b200.h."""
    import re

    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|uint64_t)\s+(pg_\w+)\s*\(", txt, re.M)))


RESTYPES = {"pg_launch_count": C.c_uint64}


def _declare(lib):
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = RESTYPES.get(name, C.c_int)
