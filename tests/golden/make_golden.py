"""Regenerates the committed golden fixtures of tests/golden/ (run in the build container).

kats.json
  * Philox4x32-10 known answers of the reference's own tests (Random123 vectors,
    reference proj/tests/test_rng.cpp:10-31) and FNV-1a vectors (test_driver.cpp:41-45);
  * the reference's OWN rng.cpp (compiled from /root/reference by oracle/build_ref.sh into
    oracle/_ref/libref_rng.so): first draws of next_u32 / uniform / gaussian3 for a few
    (seed, stream) pairs, and the serialized state after a partial block (rng.cpp:76-94).
replay_<name>.npz
  * oracle trajectories (walker positions, tau, per-step estimates) of the synthetic sets,
    with the FNV-1a hash of the generated SPINOR-TEXT they were made from.

Usage: python tests/golden/make_golden.py   (needs oracle/build and oracle/_ref built)
"""
from __future__ import annotations

import ctypes as C
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import oracle_py  # noqa: E402


def ref_lib():
    L = C.CDLL(str(oracle_py.REF_LIB))
    L.ref_philox_block.argtypes = [C.POINTER(C.c_uint32)] * 3
    L.ref_philox_stream.argtypes = [C.c_uint64, C.c_uint32, C.c_int, C.c_int, C.POINTER(C.c_double)]
    L.ref_philox_state.argtypes = [C.c_uint64, C.c_uint32, C.c_int, C.c_char_p, C.c_int]
    return L


def main():
    kats = {
        "source": "reference proj/tests/test_rng.cpp:10-31 (Random123 kat_vectors), test_driver.cpp:41-45",
        "philox_block": [
            {"ctr": [0, 0, 0, 0], "key": [0, 0], "out": [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]},
            {"ctr": [0xFFFFFFFF] * 4, "key": [0xFFFFFFFF] * 2,
             "out": [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]},
            {"ctr": [0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], "key": [0xA4093822, 0x299F31D0],
             "out": [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]},
        ],
        "fnv1a64": [["", 0xCBF29CE484222325], ["a", 0xAF63DC4C8601EC8C], ["foobar", 0x85944171F73967E8]],
    }
    R = ref_lib()
    streams = []
    for seed, stream in [(42, 0), (42, 1), (7, 3), (0x4C4C, 0), (2**40 + 5, 9)]:
        rec = {"seed": seed, "stream": stream}
        for kind, name, n in [(0, "u32", 24), (1, "uniform", 16), (2, "gaussian3", 8)]:
            out = (C.c_double * (3 * n))()
            R.ref_philox_stream(seed, stream, kind, n, out)
            vals = list(out)[: (3 * n if kind == 2 else n)]
            rec[name] = [int(v) for v in vals] if kind == 0 else [float.hex(v) for v in vals]
        buf = C.create_string_buffer(256)
        R.ref_philox_state(seed, stream, 5, buf, 256)
        rec["state_after_5_u32"] = buf.value.decode()
        streams.append(rec)
    kats["reference_rng_cpp_streams"] = streams
    (HERE / "kats.json").write_text(json.dumps(kats, indent=1))

    from paper_2203_05632_b200 import generate_config
    from paper_2203_05632_b200 import native
    with tempfile.TemporaryDirectory() as d:
        # (fixture, generator config, walkers, burn-in, steps, step size, estimator)
        for tag, name, m, burn, nsteps, step, phys in [
                ("cfg1", "cfg1", 16, 50, 12, 0.3, False), ("syn1c", "syn1c", 6, 50, 12, 0.0, False),
                ("syn2c", "syn2c", 5, 50, 12, 0.0, False), ("cfg2", "cfg2", 12, 30, 3, 0.0, False),
                ("cfg3", "cfg3", 10, 20, 2, 0.0, False), ("cfg4", "cfg4", 6, 10, 1, 0.0, False),
                ("cfg2_physical", "cfg2", 12, 30, 3, 0.0, True)]:
            sp, conf = generate_config(name, d)
            raw = sp.read_bytes()
            fnv = native.host().mcmp2h_fnv1a64(raw, len(raw))
            text = conf.read_text() + ("estimator physical\n" if phys else "")
            orc = oracle_py.OracleSystem(sp, text)
            tr = orc.trajectory(seed=3, stream=0, m=m, burn=burn, nsteps=nsteps, step_size=step, adapt=step == 0.0,
                                physical=phys)
            np.savez_compressed(HERE / f"replay_{tag}.npz", walkers=tr["walkers"], tau=tr["tau"], est=tr["est"],
                                init=tr["init"], spinor_fnv1a=np.uint64(fnv), m=m, step_size=step,
                                config=name, physical=phys)
    print("wrote", sorted(p.name for p in HERE.iterdir()))


if __name__ == "__main__":
    main()
