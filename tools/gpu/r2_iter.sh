set -u
O=gpurun_out
T=${TAG:-r2r}
timeout 900 python -m pytest tests/test_gpu_oz.py tests/test_gpu_guard.py -x -q > $O/${T}_pytest.log 2>&1; echo "pytest exit $?" >> $O/${T}_pytest.log
timeout 600 python tools/guard_cost.py cfg4 256 2e-10 > $O/${T}_guard_cost.json 2> $O/${T}_guard_cost.err
make -C paper_2203_05632_b200/csrc OUT=../lib_tl OBJ=build_tl EXTRA_NVFLAGS=-DOZ_TIMELINE > $O/${T}_tl_build.log 2>&1 && cp paper_2203_05632_b200/lib/libmcmp2host.so paper_2203_05632_b200/lib_tl/
MCMP2_LIBDIR=paper_2203_05632_b200/lib_tl timeout 300 python tools/oz_timeline.py cfg4 > $O/${T}_timeline.json 2> $O/${T}_timeline.err
