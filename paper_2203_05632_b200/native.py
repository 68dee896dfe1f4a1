"""ctypes bindings of the in-tree native libraries.

lib/libmcmp2dev.so   the sm_100a walker loop behind include/mcmp2dev.h (the drop-in C ABI)
lib/libmcmp2host.so  the C++ host driver behind include/mcmp2host.h

Nothing here computes: every call goes to the native libraries, and loading fails loudly
when they are missing (there is no CPU fallback for the walker loop).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

PKG = Path(__file__).resolve().parent
LIB = Path(os.environ.get("MCMP2_LIBDIR", PKG / "lib"))  # override only for kernel-variant experiments

OK, INVALID_ARGUMENT, RUNTIME, CUDA = 0, 1, 2, 3


class Mcmp2Error(RuntimeError):
    """Raised for MCMP2DEV_RUNTIME / MCMP2DEV_CUDA (reference std::runtime_error)."""


class Mcmp2ArgumentError(ValueError):
    """Raised for MCMP2DEV_INVALID_ARGUMENT (reference std::invalid_argument)."""


class Ensemble(C.Structure):  # mcmp2dev_ensemble
    _fields_ = [
        ("m", C.c_int),
        ("sigma_step", C.c_double),
        ("proposed", C.c_longlong),
        ("accepted", C.c_longlong),
        ("rng_key", C.c_uint32 * 2),
        ("rng_counter", C.c_uint32 * 4),
        ("rng_idx", C.c_uint32),
        ("walkers", C.POINTER(C.c_double)),
    ]


class Step(C.Structure):  # mcmp2dev_step
    _fields_ = [(n, C.c_double) for n in
                ("value", "imag", "direct_re", "direct_im", "exchange_re", "exchange_im")]


class StepEx(C.Structure):  # mcmp2dev_step_ex
    _fields_ = [(n, C.c_double) for n in
                ("value", "imag", "direct_re", "direct_im", "exchange_re", "exchange_im",
                 "est_err_direct", "est_err_exchange", "abs_direct", "abs_exchange")] + \
               [("int8_v", C.c_int), ("fallback", C.c_int)]


_dev = None
_host = None


def _load(name: str) -> C.CDLL:
    path = LIB / name
    if not path.exists():
        raise ImportError(f"{path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(make -C paper_2203_05632_b200); there is no CPU fallback")
    return C.CDLL(str(path), mode=C.RTLD_GLOBAL)


def dev() -> C.CDLL:
    global _dev
    if _dev is None:
        d = _load("libmcmp2dev.so")
        vp, dp, ip = C.c_void_p, C.POINTER(C.c_double), C.c_int
        d.mcmp2dev_last_error.restype = C.c_char_p
        d.mcmp2dev_last_error.argtypes = [vp]
        d.mcmp2dev_create.argtypes = [vp, ip, ip, C.POINTER(vp)]
        d.mcmp2dev_destroy.argtypes = [vp]
        d.mcmp2dev_init_ensemble.argtypes = [vp, ip, C.c_uint64, C.c_uint32]
        d.mcmp2dev_burn_in.argtypes = [vp, C.c_long, ip]
        d.mcmp2dev_set_sigma_step.argtypes = [vp, C.c_double]
        d.mcmp2dev_set_ensemble.argtypes = [vp, C.POINTER(Ensemble)]
        d.mcmp2dev_get_ensemble.argtypes = [vp, C.POINTER(Ensemble)]
        d.mcmp2dev_advance.argtypes = [vp, C.c_long, dp, dp]
        d.mcmp2dev_replay.argtypes = [vp, ip, C.c_long, dp, dp, C.POINTER(Step)]
        d.mcmp2dev_profile.argtypes = [vp, ip, ip, dp]
        d.mcmp2dev_work.argtypes = [vp, dp, dp, dp]
        d.mcmp2dev_synchronize.argtypes = [vp]
        d.mcmp2dev_stream.restype = vp
        d.mcmp2dev_stream.argtypes = [vp]
        d.mcmp2dev_abi_version.restype = ip
        d.mcmp2dev_kramers.argtypes = [vp, ip]
        d.mcmp2dev_pair_path.argtypes = [vp, ip]
        d.mcmp2dev_profile_pair.argtypes = [vp, dp]
        d.mcmp2dev_oz_truncation.argtypes = [vp, ip]
        d.mcmp2dev_oz_ksteps.argtypes = [vp, dp]
        d.mcmp2dev_oz_overlap.argtypes = [vp, ip]
        d.mcmp2dev_work_executed.argtypes = [vp, dp]
        d.mcmp2dev_prepare.argtypes = [vp]
        d.mcmp2dev_init_batch.argtypes = [vp, ip, ip, C.c_uint64, C.c_uint32]
        d.mcmp2dev_batch_size.argtypes = [vp]
        d.mcmp2dev_get_ensemble_at.argtypes = [vp, ip, C.POINTER(Ensemble)]
        d.mcmp2dev_set_ensemble_at.argtypes = [vp, ip, C.POINTER(Ensemble)]
        d.mcmp2dev_get_ensembles.argtypes = [vp, C.POINTER(Ensemble)]
        d.mcmp2dev_set_ensembles.argtypes = [vp, C.POINTER(Ensemble)]
        d.mcmp2dev_advance_batch.argtypes = [vp, C.c_long, ip, dp, dp]
        d.mcmp2dev_advance_ex.argtypes = [vp, C.c_long, C.POINTER(StepEx)]
        d.mcmp2dev_replay_ex.argtypes = [vp, ip, C.c_long, dp, dp, C.POINTER(StepEx)]
        d.mcmp2dev_guard.argtypes = [vp, C.c_double, dp]
        d.mcmp2dev_guard_stats.argtypes = [vp, dp]
        d.mcmp2dev_kramers_deviation.argtypes = [vp, dp]
        _dev = d
    return _dev


def host() -> C.CDLL:
    global _host
    if _host is None:
        dev()
        h = _load("libmcmp2host.so")
        vp, cp, ip, dp = C.c_void_p, C.c_char_p, C.c_int, C.POINTER(C.c_double)
        h.mcmp2h_last_error.restype = cp
        h.mcmp2h_run.argtypes = [cp, cp, ip]
        h.mcmp2h_run_hooked.argtypes = [cp, C.c_long, cp, ip]
        h.mcmp2h_resume.argtypes = [cp, cp, ip]
        h.mcmp2h_merge.argtypes = [C.POINTER(cp), ip, dp, dp, C.POINTER(C.c_longlong)]
        h.mcmp2h_parse_config.argtypes = [cp, cp, ip]
        h.mcmp2h_fnv1a64.restype = C.c_uint64
        h.mcmp2h_fnv1a64.argtypes = [cp, C.c_long]
        h.mcmp2h_system_load.restype = vp
        h.mcmp2h_system_load.argtypes = [cp, cp]
        h.mcmp2h_system_free.argtypes = [vp]
        h.mcmp2h_system_view.restype = vp
        h.mcmp2h_system_view.argtypes = [vp]
        h.mcmp2h_system_info.argtypes = [vp, C.POINTER(C.c_int), dp]
        h.mcmp2h_system_g.argtypes = [vp, dp, ip, dp]
        h.mcmp2h_save_spinor_set.argtypes = [cp, cp]
        h.mcmp2h_worker_create.restype = vp
        h.mcmp2h_worker_create.argtypes = [cp, ip, ip]
        h.mcmp2h_worker_free.argtypes = [vp]
        h.mcmp2h_worker_advance.argtypes = [vp, C.c_long, dp, dp]
        h.mcmp2h_worker_stats.argtypes = [vp, dp]
        h.mcmp2h_worker_block_means.argtypes = [vp, dp, ip]
        h.mcmp2h_worker_device.restype = vp
        h.mcmp2h_worker_device.argtypes = [vp]
        lp = C.POINTER(C.c_long)
        h.mcmp2h_group_create.restype = vp
        h.mcmp2h_group_create.argtypes = [cp, ip, ip, ip]
        h.mcmp2h_group_resume.restype = vp
        h.mcmp2h_group_resume.argtypes = [cp, ip, ip, ip]
        h.mcmp2h_group_free.argtypes = [vp]
        h.mcmp2h_group_size.argtypes = [vp]
        h.mcmp2h_group_advance.argtypes = [vp, C.POINTER(C.c_longlong)]
        h.mcmp2h_group_stats.argtypes = [vp, ip, dp]
        h.mcmp2h_group_record.argtypes = [vp, ip, cp, C.c_long, lp]
        h.mcmp2h_group_trace.argtypes = [vp, ip, cp, C.c_long, lp]
        h.mcmp2h_checkpoint_header.argtypes = [cp, ip, cp, C.c_long, lp]
        h.mcmp2h_checkpoint_config.argtypes = [cp, cp, ip, C.POINTER(C.c_int)]
        h.mcmp2h_merge_estimates.argtypes = [dp, ip, dp]
        h.mcmp2h_blocking.argtypes = [dp, C.c_long, C.c_long, dp]
        h.mcmp2h_config_hash.restype = C.c_uint64
        h.mcmp2h_config_hash.argtypes = [cp, C.c_uint64]
        h.mcmp2h_philox_stream.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, ip, C.POINTER(C.c_uint32)]
        h.mcmp2h_generate.argtypes = [cp, cp]
        _host = h
    return _host


def dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


def check_dev(rc: int, handle=None) -> None:
    if rc == OK:
        return
    msg = dev().mcmp2dev_last_error(handle).decode()
    if rc == INVALID_ARGUMENT:
        raise Mcmp2ArgumentError(msg)
    raise Mcmp2Error(msg)


def check_host(rc: int) -> None:
    if rc == 0:
        return
    msg = host().mcmp2h_last_error().decode()
    if rc == 1:
        raise Mcmp2ArgumentError(msg)
    raise Mcmp2Error(msg)


def exported_symbols(header: Path) -> list[str]:
    """Function names declared in a C header of include/ (for the ABI export test)."""
    import re
    text = header.read_text()
    return sorted(set(re.findall(r"\b(mcmp2(?:dev|h)_[a-z0-9_]+)\s*\(", text)))


def repo_root() -> Path:
    return Path(os.environ.get("GRAFT_REPO_ROOT", PKG.parent))
