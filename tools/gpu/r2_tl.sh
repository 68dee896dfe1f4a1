set -u
O=gpurun_out
make -C paper_2203_05632_b200/csrc OUT=../lib_tl OBJ=build_tl EXTRA_NVFLAGS=-DOZ_TIMELINE > $O/r2i_tl_build.log 2>&1 && cp paper_2203_05632_b200/lib/libmcmp2host.so paper_2203_05632_b200/lib_tl/
MCMP2_LIBDIR=paper_2203_05632_b200/lib_tl timeout 300 python tools/oz_timeline.py cfg4 > $O/r2i_timeline_cfg4.json 2> $O/r2i_timeline_cfg4.err
