"""ctypes binding of libboba_b200.so (the C ABI in include/boba_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2306_10410_b200/csrc``).  There is deliberately no fallback:
if the library is missing, importing this module raises, and every compute
entry point needs a CUDA device (the kernels are sm_100a only).
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BOBA_LIB_PATH") or os.path.join(_HERE, "libboba_b200.so")  # override: experiments only
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "boba_b200.h")

BOBA_OK, BOBA_EINVAL, BOBA_ECUDA, BOBA_ERANGE, BOBA_ENOMEM = 0, 1, 2, 3, 4
UNSET_U32 = 0xFFFFFFFF

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(there is no CPU fallback for the BOBA hot path)"
    )

lib = ctypes.CDLL(LIB_PATH)

_P = ctypes.c_void_p
_U64 = ctypes.c_uint64
_U32 = ctypes.c_uint32
_I = ctypes.c_int
_D = ctypes.c_double
_SZ = ctypes.c_size_t

# name -> (argtypes, restype); mirrors include/boba_b200.h one to one.
SIGNATURES = {
    "boba_abi_version": ([], _I),
    "boba_last_error": ([], ctypes.c_char_p),
    "boba_first_occurrence": ([_P, _P, _U64, _U32, _P, _I, _P], _I),
    "boba_first_occurrence_workspace_size": ([], _SZ),
    "boba_first_occurrence_shard_workspace_size": ([_U32], _SZ),
    "boba_first_occurrence_shard": ([_P, _P, _U64, _U64, _U64, _U32, _P, _I, _P, _SZ, _P], _I),
    "boba_compact_workspace_size": ([_U64, _U32], _SZ),
    "boba_compact": ([_P, _U64, _U32, _P, _P, _P, _P, _SZ, _P], _I),
    "boba_order_workspace_size": ([_U64, _U32], _SZ),
    "boba_order": ([_P, _P, _U64, _U32, _I, _P, _P, _P, _P, _SZ, _P], _I),
    "boba_relabel": ([_P, _P, _U64, _U32, _P, _P, _P, _P, _P], _I),
    "boba_degrees": ([_P, _U64, _U32, _P, _P], _I),
    "boba_coo_to_csr_workspace_size": ([_U64, _U32, _I], _SZ),
    "boba_coo_to_csr": ([_P, _P, _P, _U64, _U32, _P, _P, _P, _P, _P, _SZ, _P], _I),
    "boba_coo_to_csr_ex": ([_P, _P, _P, _U64, _U32, _P, _P, _P, _P, _P, _SZ, _I, _P], _I),
    "boba_coo_to_csr_first_hist": ([_P, _U64, _U32, _P, _SZ, _P], _I),
    "boba_spmv_workspace_size": ([_U32, _U64], _SZ),
    "boba_spmv": ([_P, _P, _P, _P, _P, _U32, _U64, _P, _SZ, _P], _I),
    "boba_spmv_f64": ([_P, _P, _P, _P, _P, _U32, _U64, _P, _SZ, _P], _I),
    "boba_spmv_ex": ([_P, _P, _P, _P, _P, _U32, _U64, _P, _SZ, _I, _P], _I),
    "boba_spmv_f64_ex": ([_P, _P, _P, _P, _P, _U32, _U64, _P, _SZ, _I, _P], _I),
    "boba_reorder_to_csr_workspace_size": ([_U64, _U32, _I], _SZ),
    "boba_reorder_to_csr": ([_P, _P, _P, _U64, _U32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P], _I),
    "boba_reorder_to_csr_timed": ([_P, _P, _P, _U64, _U32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P, _P], _I),
    "boba_ctx_create": ([_U64, _U32, ctypes.POINTER(_P)], _I),
    "boba_ctx_destroy": ([_P], None),
    "boba_ctx_reorder_to_csr_host": ([_P, _P, _P, _U64, _U32, _P, _P, _P, _P, _P, _P], _I),
    "boba_ctx_submit_host": ([_P, _P, _P, _U64, _U32, _P, _P, _P, _P, _P, _P, ctypes.POINTER(_U64)], _I),
    "boba_ctx_wait": ([_P, _U64], _I),
    "boba_nbr_workspace_size": ([_U64, _U32], _SZ),
    "boba_nbr": ([_P, _P, _U32, _U64, _U32, _P, _P, _SZ, _P], _I),
    "boba_compact_relabel_workspace_size": ([_U64, _U32], _SZ),
    "boba_compact_relabel": ([_P, _U64, _U32, _P, _P, _U64, _P, _P, _P, _P, _P, _SZ, _P], _I),
    "boba_range_partition_ex": ([_P, _P, _U64, _P, _I, _I, _P, _P, _P, _P, _SZ, _P], _I),
    "boba_compact_shard_workspace_size": ([_U64, _U32], _SZ),
    "boba_compact_shard_mark": ([_P, _U32, _U64, _U64, _U64, _P, _P, _SZ, _P], _I),
    "boba_compact_shard_assign": ([_P, _U32, _U64, _U64, _U64, _P, _I, _I, _P, _P, _SZ, _P], _I),
    "boba_hub_table_bytes": ([], _SZ),
    "boba_order_from_label": ([_P, _U32, _P, _P, _P], _I),
    "boba_relabel_hubs": ([_P, _P, _U64, _U32, _P, _P, _P, _P, _P], _I),
    "boba_row_cut_buckets": ([_U32], _U32),
    "boba_row_cut_hist": ([_P, _U64, _U32, _P, _P], _I),
    "boba_row_cut": ([_P, _P, _U32, _U64, _I, _P, _P], _I),
    "boba_sharded_workspace_size": ([_U64, _U32, _I, _U64], _SZ),
    "boba_sharded_reorder_to_csr_nccl": ([_P, _P, _U64, _U64, _U64, _U32, _P, _P, _P, _P, _P, _P, _P, _P, _U64, _P,
                                          _P, _P, _SZ, _P], _I),
    "boba_reorder_to_csr_graph_create": ([_P, _P, _U64, _U32, _P, _P, _P, _P, _P, _P, _P, _P, _SZ,
                                          ctypes.POINTER(_P)], _I),
    "boba_reorder_to_csr_graph_create_timed": ([_P, _P, _U64, _U32, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P,
                                                ctypes.POINTER(_P)], _I),
    "boba_graph_launch": ([_P, _P], _I),
    "boba_reorder_to_csr_graph_destroy": ([_P], None),
    "boba_graph_kernel_nodes": ([_P, _P], _I),
    "boba_narrow_ids": ([_P, _U64, _U64, _P, ctypes.POINTER(ctypes.c_int64), _P], _I),
    "boba_host_to_device_ids": ([_P, _U64, _U64, _P, ctypes.POINTER(ctypes.c_int64), _P], _I),
    "boba_device_to_host_ids": ([_P, _U64, _P, _P], _I),
    "boba_device_to_host_ranks": ([_P, _U64, _P, _P], _I),
    "boba_widen_ids": ([_P, _U64, _P, _P], _I),
    "boba_exclusive_scan_workspace_size": ([_U64], _SZ),
    "boba_exclusive_scan_u32": ([_P, _U32, _P, _P, _SZ, _P], _I),
    "boba_bias_u32": ([_P, _U64, _P, _P], _I),
    "boba_offset_ids": ([_P, _U64, _U32, _P, _P], _I),
    "boba_range_partition_workspace_size": ([_U64, _I], _SZ),
    "boba_range_partition": ([_P, _P, _U64, _P, _I, _P, _P, _P, _P, _SZ, _P], _I),
    "boba_gather_u32": ([_P, _P, _U64, _P, _P], _I),
    "boba_total_degrees": ([_P, _P, _U64, _U32, _P, _P], _I),
    "boba_degree_order_workspace_size": ([_U64, _U32], _SZ),
    "boba_degree_order": ([_P, _P, _U64, _U32, _P, _P, _P, _SZ, _P], _I),
    "boba_hub_order": ([_P, _P, _U64, _U32, _P, _P, _P, _SZ, _P], _I),
    "boba_sort_coo_by_destination_workspace_size": ([_U64, _U32], _SZ),
    "boba_sort_coo_by_destination": ([_P, _P, _P, _U64, _U32, _P, _P, _P, _P, _SZ, _P], _I),
    "boba_pagerank_workspace_size": ([_U32, _U64], _SZ),
    "boba_pagerank": ([_P, _P, _P, _U32, _U64, _D, _D, _I, _P, _P, _P, _SZ, _P], _I),
    "boba_generate_rmat": ([_I, _U64, _U64, _P, _P, _P], _I),
    "boba_generate_rmat_range": ([_I, _U64, _U64, _U64, _P, _P, _P], _I),
    "boba_generate_grid": ([_U32, _U32, _P, _P, _P], _I),
}

for _name, (_args, _res) in SIGNATURES.items():
    _fn = getattr(lib, _name)
    _fn.argtypes = _args
    _fn.restype = _res


class NativeError(RuntimeError):
    """A libboba_b200 call failed (CUDA error or invalid argument)."""

    def __init__(self, code: int, message: str):
        super().__init__(f"[boba_b200 error {code}] {message}")
        self.code = code


def check(rc: int) -> None:
    if rc != BOBA_OK:
        msg = lib.boba_last_error()
        raise NativeError(rc, msg.decode() if msg else "unknown error")


def exported_symbols() -> list[str]:
    return list(SIGNATURES)
