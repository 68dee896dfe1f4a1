"""Timeline of oz_vgemm_kernel (main pass) from the OZ_TIMELINE debug build: per CTA and tile,
the MMA issuer's wait for the accumulators and each epilogue warp's drain and contraction, in
SM cycles. Build: make -C paper_2203_05632_b200/csrc OUT=../lib_tl OBJ=build_tl
EXTRA_NVFLAGS=-DOZ_TIMELINE && cp paper_2203_05632_b200/lib/libmcmp2host.so paper_2203_05632_b200/lib_tl/
usage: MCMP2_LIBDIR=paper_2203_05632_b200/lib_tl python tools/oz_timeline.py [cfg4] [tol] [tau]
(tol 1e-300 forces the guard's refinement pass; its stamps then overwrite the main pass's)"""
import ctypes as C
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2203_05632_b200 import DeviceWalker, System, generate_config, native  # noqa: E402

EPW, TILES, CTAS = 8, 128, 160
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
m = {"cfg3": 512, "cfg4": 2048}.get(cfg, 8192)
with tempfile.TemporaryDirectory() as d:
    sp, conf = generate_config(cfg, d)
    dw = DeviceWalker(System(sp, conf.read_text()), max_walkers=m)
    dw.guard(float(sys.argv[2]) if len(sys.argv) > 2 else 1e300)  # default: the refinement never runs
    dw.init_ensemble(m, seed=1)
    dw.burn_in(20)
    dw.advance(3)
    if len(sys.argv) > 3:  # one replayed step at a chosen tau (the k-step truncation follows it)
        dw.replay(dw.get_ensemble().walkers[:, :8][None], np.array([float(sys.argv[3])]))
    buf = np.zeros((CTAS, TILES, 3 + 3 * EPW), dtype=np.uint64)
    f = native.dev().mcmp2dev_debug_oz_timeline
    f.argtypes = [C.c_void_p, C.c_size_t]
    assert f(buf.ctypes.data, buf.nbytes) == 0
t = buf.astype(np.float64)
ctas = [b for b in range(CTAS) if t[b, 0, 1] > 0]
res = {"ctas": len(ctas)}
stall, drain, late, mma, contract, period = [], [], [], [], [], []
for b in ctas:
    n = int(np.sum(t[b, :, 1] > 0))
    for i in range(n):
        acq, issued = t[b, i, 1], t[b, i, 2]
        full = t[b, i, 3::3][:EPW]
        rel = t[b, i, 4::3][:EPW]
        done = t[b, i, 5::3][:EPW]
        if i > 0:
            period.append(acq - t[b, i - 1, 1])
            stall.append(acq - t[b, i, 0])              # MMA issuer waiting for the accumulators
            prev_full = t[b, i - 1, 3::3][:EPW].min()
            drain.append(t[b, i - 1, 4::3][:EPW].max() - prev_full)  # MMA done -> all warps released
            late.append(max(0.0, (t[b, i - 1, 5::3][:EPW].max() if i > 1 else 0) - full.min()))
        mma.append(full.min() - acq)                    # accumulators acquired -> MMAs complete
        contract.append((done - rel).mean())
for k, v in (("tile_period", period), ("mma_issuer_stall", stall), ("drain_full_to_release", drain),
             ("mma_acquire_to_complete", mma), ("contract_per_warp", contract), ("epilogue_late", late)):
    v = np.array(v)
    res[k] = {"mean": float(v.mean()), "p50": float(np.median(v)), "p90": float(np.percentile(v, 90)), "max": float(v.max())}
print(json.dumps(res, indent=1))
