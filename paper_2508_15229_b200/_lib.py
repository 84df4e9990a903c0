"""ctypes binding of the C-ABI in include/svt.h (libsvt.so, sm_100a CUDA).

There is no CPU fallback: importing this module fails loudly when the
shared library is missing, and every compute call raises ``Error`` when no
CUDA device is usable. Status codes map onto the reference's exception
taxonomy (/root/reference/proj/include/subvocab/error.hpp:10-38).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(HERE, "lib")
LIB_PATH = os.path.join(LIB_DIR, "libsvt.so")

SVT_F32, SVT_F16, SVT_BF16 = 0, 1, 2
SVT_WEIGHTS_STABLE = 1  # svt.h: rows not written by the kernel a launch depends on
SVT_ROWS_HIDDEN_STABLE = 2  # svt.h: h not written by it either (rows_hs_kernel)
GROUP_ROWS = 32
GROUP_META_BYTES = 32


class Error(RuntimeError):
    """subvocab::Error (exit code 1) — also CUDA/runtime failures."""

    exit_code = 1


class ConfigError(Error):
    exit_code = 2


class ParseError(Error):
    exit_code = 3


class IntegrityError(Error):
    exit_code = 4


_ERRORS = {1: Error, 2: ConfigError, 3: ParseError, 4: IntegrityError}

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA extension first "
        "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")

lib = C.CDLL(LIB_PATH)

_vp, _sz, _i32, _i64, _u32, _u64 = C.c_void_p, C.c_size_t, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64

_SIGS = {
    "svt_abi_version": ([], C.c_int),
    "svt_last_error": ([], C.c_char_p),
    "svt_device_count": ([], C.c_int),
    "svt_dtype_size": ([C.c_int], _sz),
    "svt_set_device": ([C.c_int], C.c_int),
    "svt_get_device": ([C.POINTER(C.c_int)], C.c_int),
    "svt_device_alloc": ([C.POINTER(_vp), _sz], C.c_int),
    "svt_device_free": ([_vp], C.c_int),
    "svt_host_alloc_pinned": ([C.POINTER(_vp), _sz], C.c_int),
    "svt_host_free_pinned": ([_vp], C.c_int),
    "svt_memcpy_h2d": ([_vp, _vp, _sz, _vp], C.c_int),
    "svt_memcpy_d2h": ([_vp, _vp, _sz, _vp], C.c_int),
    "svt_memcpy_d2d": ([_vp, _vp, _sz, _vp], C.c_int),
    "svt_memset": ([_vp, C.c_int, _sz, _vp], C.c_int),
    "svt_stream_create": ([C.POINTER(_vp)], C.c_int),
    "svt_stream_destroy": ([_vp], C.c_int),
    "svt_stream_synchronize": ([_vp], C.c_int),
    "svt_set_tuning": ([C.c_int, C.c_int], None),
    "svt_set_debug": ([_vp], None),
    "svt_head_random": ([_vp, C.c_int, C.c_int, _u64, _u64, _u64, _vp], C.c_int),
    "svt_convert_from_f32": ([_vp, _vp, C.c_int, _u64, _vp], C.c_int),
    "svt_convert_to_f32": ([_vp, C.c_int, _vp, _u64, _vp], C.c_int),
    "svt_select_batched": ([_vp, _sz, _sz, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
                           C.c_int),
    "svt_bitset_insert": ([_vp, _sz, _sz, _vp, _vp, _vp], C.c_int),
    "svt_union_plans": ([_vp, _vp, _i32, _sz, _vp, _vp, _vp, _vp, _vp], C.c_int),
    "svt_plan_layout": ([_vp, _vp, _i32, _vp, _vp, _i64, _vp], C.c_int),
    "svt_gather_plans": ([_vp, C.c_int, _sz, _sz, _vp, _vp, _vp, _i32, _i64, _vp, _vp, _vp],
                         C.c_int),
    "svt_gather_rows": ([_vp, C.c_int, _sz, _sz, _vp, _sz, _vp, _vp, _vp], C.c_int),
    "svt_subhead_bytes": ([C.c_int, _sz, _i64], _sz),
    "svt_gather_interleaved": ([_vp, C.c_int, _sz, _sz, _vp, _vp, _vp, _i32, _i64, _vp, _vp, _vp],
                               C.c_int),
    "svt_logits": ([_vp, C.c_int, _sz, _sz, _vp, _vp, _vp], C.c_int),
    "svt_logits_rows": ([_vp, C.c_int, _sz, _sz, _vp, _vp, _vp, _i32, _i64, _vp, _sz, _vp, _vp,
                         _vp], C.c_int),
    "svt_logits_interleaved": ([_vp, C.c_int, _sz, _vp, _vp, _i32, _i64, _vp, _sz, _vp, _vp, _vp],
                               C.c_int),
    "svt_greedy_step": ([_vp, C.c_int, _sz, _sz, _vp, _vp, _vp, _vp, _vp, _vp], C.c_int),
    "svt_greedy_workspace_bytes": ([_i32, _i64], _sz),
    "svt_greedy_interleaved": ([_vp, C.c_int, _sz, _vp, _vp, _vp, _i32, _i64, _vp, _sz, _u32, _i32,
                                _i32, _vp, _vp, _vp, _vp, _vp], C.c_int),
    "svt_greedy_fused": ([_vp, C.c_int, _sz, _sz, _vp, _vp, _vp, _i32, _i64, _vp, _sz, _u32, _i32,
                          _i32, _vp, _vp, _vp, _vp, _vp], C.c_int),
    "svt_certified_workspace_bytes": ([_i32, _i64], _sz),
    "svt_greedy_certified": ([_vp, C.c_int, _sz, _vp, _vp, _vp, _i32, _i64, _vp, _sz, _vp, _vp,
                              _vp, _vp], C.c_int),
    "svt_greedy_rows_workspace_bytes": ([_sz], _sz),
    "svt_rows_set_debug": ([_vp], None),
    "svt_greedy_certified_rows": ([_vp, C.c_int, _sz, _sz, _vp, _sz, _vp, _vp, _u32, _i32, _i32,
                                   _vp, _vp, _vp, _vp, _vp], C.c_int),
    "svt_prefill_workspace_bytes": ([_i32, _i32], _sz),
    "svt_prefill_score": ([_vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _vp, _vp,
                           _vp, _vp], C.c_int),
    "svt_prefill_score_fused": ([_vp, _vp, _i64, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _vp, _vp,
                                 _vp, _vp], C.c_int),
    "svt_prefill_static_pad": ([_i64], _i64),
    "svt_prefill_split_plans": ([_vp, _vp, _vp, _i32, _vp, C.c_size_t, _vp, _i64, _vp, _vp, _vp,
                                 _vp, _vp, _vp, _vp], C.c_int),
    "svt_prefill_score_split": ([_vp, _vp, _i64, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _i32,
                                 _i32, _i32, _vp, _vp, _vp, _vp], C.c_int),
    "svt_decode_split_plans": ([_vp, _vp, _vp, _i32, _vp, _sz, _vp, _i64, _vp, _vp, _vp, _vp,
                                _vp, _vp], C.c_int),
    "svt_greedy_split_workspace_bytes": ([_i32, _i64, _i64, _sz], _sz),
    "svt_greedy_split": ([_vp, C.c_int, _i64, _sz, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                          _i32, _i64, _vp, _sz, _i32, _vp, _vp, _vp, _vp], C.c_int),
    "svt_row_norms_bf16": ([_vp, _i64, _i32, _vp, _vp], C.c_int),
    "svt_prefill_set_tuning": ([_i32, _i32], C.c_int),
    "svt_prefill_get_tuning": ([_vp, _vp], None),
    "svt_prefill_effective_nsplit": ([_i32, _i32], _i32),
    "svt_prefill_offsets": ([_i32, _i32, _vp], None),
    "svt_prefill_meta_offset": ([_i32, _i32], _i64),
    "svt_shard_combine": ([_vp, _i32, _i32, _vp, _vp, _vp], C.c_int),
    "svt_topk_logits": ([_vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _vp, _vp, _vp], C.c_int),
    "svt_sharded_workspace_bytes": ([_sz, _i32], _sz),
    "svt_sharded_greedy": ([_vp, C.c_int, _sz, _sz, _vp, _sz, _vp, _vp, _u32, _i32, _vp, _i32,
                            _vp, _vp, _vp, _vp], C.c_int),
    "svt_nccl_get_unique_id": ([_vp, _sz], C.c_int),
    "svt_nccl_comm_init": ([C.POINTER(_vp), _i32, _i32, _vp], C.c_int),
    "svt_nccl_comm_destroy": ([_vp], C.c_int),
    "svt_embed_lookup_zero_copy": ([_vp, C.c_int, _sz, _sz, _vp, _sz, _vp, _vp, _vp], C.c_int),
    "svt_embed_lookup_staged": ([_vp, C.c_int, _sz, _sz, _vp, _sz, _vp, _vp, _vp], C.c_int),
    "svt_session_create": ([C.POINTER(_vp), _vp, C.c_int, _sz, _sz, _i32, _i64, _vp], C.c_int),
    "svt_session_destroy": ([_vp], C.c_int),
    "svt_session_prepare_host": ([_vp, _vp, _sz, _vp, _vp, _i32], C.c_int),
    "svt_session_prepare_host_many": ([_vp, C.c_int32, _vp, _sz, _vp, _vp, _vp], C.c_int),
    "svt_session_plans_host": ([_vp, _vp, _vp, _vp, _vp, _vp], C.c_int),
    "svt_session_greedy_host": ([_vp, _vp, _sz, _vp, _vp], C.c_int),
    "svt_session_greedy_device": ([_vp, _vp, _sz, _vp, _vp], C.c_int),
    "svt_session_stream": ([_vp], _vp),
    "svt_session_decode_host": ([_vp, C.c_int32, _vp, C.c_int32, _vp], C.c_int),
    "svt_plan_to_json": ([_vp, _sz, _sz, _sz, _sz, _i32, _vp, _sz, _vp], C.c_int),
    "svt_plans_to_jsonl": ([_vp, _vp, _vp, _vp, _vp, _i32, _sz, _vp, _sz, _vp], C.c_int),
    "svt_plan_from_json": ([C.c_char_p, _sz, C.c_char_p, _vp, _sz, _vp, _vp, _vp, _vp], C.c_int),
    "svt_tolerance_filter": ([_vp, _vp, _sz, _vp, _sz, _i64, C.c_double, _vp, _vp, _vp, _vp,
                              _vp], C.c_int),
    "svt_profile_batch": ([_sz, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                           _vp], C.c_int),
    "svt_profile_merge": ([_sz, _vp, _vp, _vp, _vp, _vp, _vp, _vp], C.c_int),
    "svt_memory_report": ([_sz, _sz, C.c_int, _sz, _vp], C.c_int),
    "svt_simulate": ([C.c_double, C.c_double, C.c_double, _sz, _sz, C.c_int, _sz, C.c_double,
                      _vp], C.c_int),
    "svt_breakeven_rows": ([C.c_double, C.c_double, C.c_double, _sz, C.c_int, _sz, C.c_double,
                            _vp], C.c_int),
}

EXPORTED = tuple(_SIGS)

for _name, (_args, _res) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.argtypes = _args
    _fn.restype = _res


def last_error() -> str:
    m = lib.svt_last_error()
    return m.decode() if m else ""


def check(status: int, what: str = "") -> None:
    if status:
        cls = _ERRORS.get(status, Error)
        raise cls(f"{what}: {last_error()}" if what else last_error())


def call(name: str, *args) -> None:
    check(getattr(lib, name)(*args), name)
