"""B200-native MC-MP2 walker loop (arXiv 2203.05632) behind the reference's driver interface.

Layout:
  csrc/      sm_100a CUDA kernels + the C ABI (include/mcmp2dev.h) -> lib/libmcmp2dev.so
  host/      C++ host driver: SPINOR-TEXT, RunConfig, Engine, checkpoint, CLI -> lib/libmcmp2host.so, lib/mcmp2
  native.py  ctypes bindings (fail loudly when the libraries are missing)
  walker.py  Python mirror of the reference's per-worker interface over the C ABI
  distributed.py  one process per GPU, torch.distributed merge of per-worker estimates
"""
from .walker import DeviceWalker, System, generate_config, run_config_text  # noqa: F401
