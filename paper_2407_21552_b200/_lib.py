"""ctypes binding of the C ABI in include/pdm_b200.h (lib/libpdm_b200.so).

There is no CPU fallback: every compute entry point of the package goes
through this library, and ``lib()`` raises if the shared library is missing
or no CUDA device is visible.  Status codes map to Python exceptions the way
the reference's callers expect: PDM_EINVAL -> ValueError,
PDM_ECUDA / PDM_EUNSUPPORTED -> RuntimeError.
"""

from __future__ import annotations

import ctypes
from pathlib import Path

import os

# PDM_LIB_PATH: an A/B build of the same library (tools/exp/build_variant.py)
LIB_PATH = Path(os.environ.get("PDM_LIB_PATH") or
                Path(__file__).resolve().parent / "lib" / "libpdm_b200.so")

PDM_OK, PDM_EINVAL, PDM_ECUDA, PDM_EUNSUPPORTED = 0, 1, 2, 3

_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_INT = ctypes.c_int
_F64 = ctypes.c_double

# name -> argtypes (all return int status unless listed in _RESTYPES)
_SIGNATURES = {
    "pdm_version": [],
    "pdm_last_error": [],
    "pdm_device_sm_count": [_INT],
    "pdm_stream_synchronize": [_P],
    "pdm_fill_u8": [_P, _I64, _I32, _P],
    "pdm_select": [_P, _I64, _I64, _P, _I32, _I32, _P, _P],
    "pdm_select_tf": [_P, _I64, _I64, _P, _P, _P, _I32, _I32, _P, _P, _P],
    "pdm_alpha_support": [_P, _I64, _I64, _P, _P, _P],
    "pdm_combine": [_P, _I64, _I64, _I32, _P, _I32, _P, _P],
    "pdm_combine_flags": [_P, _I64, _I64, _I32, _P, _P, _P],
    "pdm_packed_chunks": [_I64],
    "pdm_count_nonlipschitz_chunks": [_P, _I64, _I64, _I32, _P, _P],
    "pdm_pack_pdms": [_P, _I64, _I64, _I32, _P, _I64, _P, _I64, _P, _P],
    "pdm_distance_transform_mask_packed": [_P, _I32, _I32, _I64, _I64, _I64, _P, _I64, _P, _I64,
                                           _P, _I64, _P, _P, _P],
    "pdm_packed_tile_bounds": [_P, _I64, _P, _I64, _I64, _I32, _P, _P],
    "pdm_merge_stats": [_P],
    "pdm_combine_packed": [_P, _I64, _P, _I64, _P, _I64, _I32, _P, _I32, _P, _P, _P],
    "pdm_combine_flags_packed": [_P, _I64, _P, _I64, _P, _I64, _I32, _P, _P, _P, _P],
    "pdm_combine_flags_auto": [_P, _I64, _P, _I64, _P, _I64, _P, _I64, _I32, _P, _P, _P, _P],
    "pdm_combine_raw_max_k": [],
    "pdm_combine_packed_to_packed": [_P, _I64, _P, _I64, _I64, _I32, _P, _I32, _P, _P, _P],
    "pdm_combine_flags_packed_to_packed": [_P, _I64, _P, _I64, _I64, _I32, _P, _P, _P, _P],
    "pdm_unpack_packed_host": [_P, _P, _I64, _P],
    "pdm_merge_packed_to_host": [_P, _I64, _P, _I64, _P, _I64, _I32, _P, _P, _I32, _P, _P, _P,
                                 _I32, _I32, _P],
    "pdm_combine_packed_host": [_P, _I64, _P, _I64, _P, _I64, _I32, _P, _P, _I32, _P, _P, _P,
                                _I32, _P],
    "pdm_gather_f64_host": [_P, _I64, _I64, _P],
    "pdm_dprime_to_host": [_P, _I64, _P, _P, _P, _I32, _I32, _P],
    "pdm_unpack_delta_host": [_P, _P, _I64, _P],
    "pdm_unpack_sparse_host": [_P, _I64, _P],
    "pdm_block_min_max": [_P, _INT, _I64, _I64, _I64, _I32, _P, _P, _P],
    "pdm_partition_mask_voxel": [_P, _INT, _I64, _I64, _I64, _I32, _P, _I32, _P, _I32, _P],
    "pdm_partition_mask_range_apron": [_P, _INT, _I64, _I64, _I64, _I32, _P, _I32, _P, _I32, _P],
    "pdm_partition_mask_minmax": [_P, _P, _INT, _I64, _P, _I32, _P, _I32, _P],
    "pdm_block_any_lut": [_P, _INT, _I64, _I64, _I64, _I32, _P, _P, _P],
    "pdm_occupancy_minmax_range": [_P, _P, _INT, _I64, ctypes.c_uint32, ctypes.c_uint32, _P, _P],
    "pdm_occupancy_minmax_prefix": [_P, _P, _INT, _I64, _P, _P, _P],
    "pdm_distance_transform": [_P, _I64, _I64, _I64, _P, _P],
    "pdm_standard_distance_map_voxel": [_P, _INT, _I64, _I64, _I64, _I32, _P, _P, _P],
    "pdm_standard_distance_map_minmax": [_P, _P, _INT, _I64, _I64, _I64, _P, _P, _P],
    "pdm_distance_transform_mask": [_P, _I32, _I32, _I64, _I64, _I64, _P, _I64, _P],
    "pdm_dt_pass_x_mask": [_P, _I32, _I32, _I64, _I64, _I64, _P, _I64, _P],
    "pdm_dt_slab_edges": [_P, _I64, _I32, _I64, _I64, _I64, _P, _P],
    "pdm_dt_slab_fold": [_P, _I64, _I32, _I64, _I64, _I64, _P, _I32, _I32, _P, _P],
    "pdm_dt_pass_yz": [_P, _I64, _I32, _I64, _I64, _I64, _P],
    "pdm_volume_range": [_P, _INT, _I64, _P, _P],
    "pdm_count_value": [_P, _I64, ctypes.c_uint32, _P, _P],
    "pdm_minmax_fold": [_P, _P, _P, _P, _INT, _I64, _P],
    "pdm_nccl_available": [],
    "pdm_nccl_unique_id": [_P],
    "pdm_nccl_comm_init": [_P, _I32, _P, _I32],
    "pdm_nccl_comm_destroy": [_P],
    "pdm_nccl_comm_count": [_P],
    "pdm_build_pdm_set_slab_nccl_workspace": [_I32, _INT, _I64, _I64, _I64, _I32, _I32],
    "pdm_build_pdm_set_slab_nccl": [_P, _P, _INT, _I64, _I64, _I64, _I32, _P, _I32, _I32, _I64,
                                    _P, _I64, _P, _I64, _P, _I64, _P, _P, _I64, _P, _P],
    "pdm_synth_volume": [_INT, _I64, _I64, _I64, _I64, _I64, _P, _I32, ctypes.c_uint64, _P, _P],
    "pdm_camera_rays": [_P, _F64, _F64, _P, _I32, _I32, _P, _P],
    "pdm_march_rays": [_P, _I32, _I64, _I64, _I64, _P, _I64, _P, _I32, _F64, _I32, _F64, _P, _P,
                       _I64, _P, _P, _P, _P, _P],
}
_RESTYPES = {"pdm_last_error": ctypes.c_char_p,
             "pdm_build_pdm_set_slab_nccl_workspace": _I64}

EXPORTED = tuple(_SIGNATURES)

_lib = None


class PdmCudaError(RuntimeError):
    """A CUDA failure or unsupported shape inside libpdm_b200."""


def load_library(path: Path | str = LIB_PATH) -> ctypes.CDLL:
    """dlopen the library and bind every exported symbol (no GPU needed)."""
    path = Path(path)
    if not path.exists():
        raise ImportError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    L = ctypes.CDLL(str(path))
    for name, argtypes in _SIGNATURES.items():
        fn = getattr(L, name)
        fn.argtypes = argtypes
        fn.restype = _RESTYPES.get(name, _INT)
    return L


def lib() -> ctypes.CDLL:
    """The bound library; raises when there is no CUDA device (no CPU fallback)."""
    global _lib
    if _lib is None:
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError(
                "paper_2407_21552_b200 runs on CUDA (sm_100a) only and no CUDA device is "
                "visible; there is no CPU fallback"
            )
        _lib = load_library()
    return _lib


def check(status: int, what: str) -> None:
    if status == PDM_OK:
        return
    msg = (_lib.pdm_last_error() or b"").decode(errors="replace") if _lib is not None else ""
    if status == PDM_EINVAL:
        raise ValueError(f"{what}: {msg}")
    raise PdmCudaError(f"{what}: {msg} (status {status})")


def stream_handle(stream=None) -> int:
    """Raw cudaStream_t of `stream` (default: torch's current stream on the
    current device; the direct accessor avoids building a Stream object)."""
    import torch

    if stream is not None:
        return int(stream.cuda_stream)
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())


def ptr(t) -> int:
    return int(t.data_ptr())
