"""Timeline of oz_vgemm_fused_kernel (the literal path's main pass, two passes per tile) from the
OZ_TIMELINE debug build: per CTA and tile, in SM cycles, the MMA issuer's waits for TMEM and the
epilogue warps' drains and contractions. Build: make -C paper_2203_05632_b200/csrc OUT=../lib_tl
OBJ=build_tl EXTRA_NVFLAGS=-DOZ_TIMELINE && cp paper_2203_05632_b200/lib/libmcmp2host.so
paper_2203_05632_b200/lib_tl/
usage: MCMP2_LIBDIR=paper_2203_05632_b200/lib_tl python tools/fz_timeline.py [cfg4]"""
import ctypes as C
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2203_05632_b200 import DeviceWalker, System, generate_config, native  # noqa: E402

EPW, TILES, CTAS, SLOTS = 8, 64, 160, 64
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
m = {"cfg3": 512, "cfg4": 2048}.get(cfg, 8192)
with tempfile.TemporaryDirectory() as d:
    sp, conf = generate_config(cfg, d)
    dw = DeviceWalker(System(sp, conf.read_text()), max_walkers=m)
    dw.guard(1e300)  # estimate only: the refinement never runs
    dw.init_ensemble(m, seed=1)
    dw.burn_in(20)
    dw.advance(3)
    buf = np.zeros((CTAS, TILES, SLOTS), dtype=np.uint64)
    f = native.dev().mcmp2dev_debug_fz_timeline
    f.argtypes = [C.c_void_p, C.c_size_t]
    assert f(buf.ctypes.data, buf.nbytes) == 0
t = buf.astype(np.float64)


def epi(b, i, k):  # stamp k (0..6) of all epilogue warps
    return t[b, i, 8 + k::7][:EPW]


ctas = [b for b in range(CTAS) if t[b, 0, 1] > 0]
keys = ["period", "mma_wait_for_tmem", "passA_mma", "passA_drain_lo", "passA_drain_hi", "passA_contract",
        "passB_wait_for_lo", "passB_mma", "passB_drain", "passB_contract_and_pairs", "epilogue_idle_before_B"]
acc = {k: [] for k in keys}
for b in ctas:
    n = int(np.sum(t[b, :, 1] > 0))
    for i in range(n):
        T = t[b, i]
        if i > 0:
            acc["period"].append(T[1] - t[b, i - 1, 1])
            acc["mma_wait_for_tmem"].append(T[1] - T[0])
        afull = epi(b, i, 0).min()
        acc["passA_mma"].append(afull - T[1])
        acc["passA_drain_lo"].append(epi(b, i, 1).max() - afull)
        acc["passA_drain_hi"].append(epi(b, i, 2).max() - epi(b, i, 1).max())
        acc["passA_contract"].append((epi(b, i, 3) - epi(b, i, 2)).mean())
        acc["passB_wait_for_lo"].append(T[3] - T[2])
        bfull = epi(b, i, 4).min()
        acc["passB_mma"].append(bfull - T[3])
        acc["passB_drain"].append(epi(b, i, 5).max() - bfull)
        acc["passB_contract_and_pairs"].append((epi(b, i, 6) - epi(b, i, 5)).mean())
        acc["epilogue_idle_before_B"].append((epi(b, i, 4) - epi(b, i, 3)).mean())
res = {"ctas": len(ctas)}
for k, v in acc.items():
    v = np.array(v)
    res[k] = {"mean": float(v.mean()), "p50": float(np.median(v)), "p90": float(np.percentile(v, 90))}
print(json.dumps(res, indent=1))
