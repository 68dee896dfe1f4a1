"""When the slice kernel and the O pass run (OZ_OVERLAP_TL debug build): first CTA start and last
CTA end of each on the global nanosecond timer over one production step, overlapped and in
series. Build: make -C paper_2203_05632_b200/csrc OUT=../lib_tl OBJ=build_tl
EXTRA_NVFLAGS=-DOZ_OVERLAP_TL && cp paper_2203_05632_b200/lib/libmcmp2host.so paper_2203_05632_b200/lib_tl/
usage: MCMP2_LIBDIR=paper_2203_05632_b200/lib_tl python tools/overlap_timeline.py [cfg4]"""
import ctypes as C
import json
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2203_05632_b200 import DeviceWalker, System, generate_config, native  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
m = {"cfg3": 512, "cfg4": 2048}.get(cfg, 8192)
fs, fo = native.dev().mcmp2dev_debug_tl_slice, native.dev().mcmp2dev_debug_tl_opass
for fn in (fs, fo):
    fn.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
bs, bo = (C.c_ulonglong * 2)(), (C.c_ulonglong * 2)()
out = {"config": cfg, "m": m}
with tempfile.TemporaryDirectory() as d:
    sp, conf = generate_config(cfg, d)
    dw = DeviceWalker(System(sp, conf.read_text()), max_walkers=m)
    dw.init_ensemble(m, seed=1)
    dw.burn_in(100)
    for mode, key in ((1, "overlap"), (0, "series")):
        dw.int8_overlap(mode)
        dw.advance(3)
        rows = []
        for _ in range(5):
            dw.synchronize()
            fs(bs, 1), fo(bo, 1)
            dw.advance(1)
            dw.synchronize()
            fs(bs, 0), fo(bo, 0)
            t0 = min(bs[0], bo[0])
            rows.append({"slice_us": [(bs[0] - t0) / 1e3, (bs[1] - t0) / 1e3],
                         "o_pass_us": [(bo[0] - t0) / 1e3, (bo[1] - t0) / 1e3]})
        out[key] = rows
print(json.dumps(out, indent=1))
