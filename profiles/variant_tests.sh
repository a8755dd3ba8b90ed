#!/bin/bash
# The GPU suite against the two compositing buffer configurations forced for
# every view (the default picks per view by pair count, so small test views
# take the big-buffer kernels and the c4 views the small-buffer ones):
#   SDGR_LIB_NAME=libsdgr_sm.so SDGR_EXTRA_FLAGS=-DSDGR_BIG_WALK_PAIRS=0 SDGR_BUILD_SUFFIX=_sm python paper_2506_21633_b200/csrc/build.py
#   SDGR_LIB_NAME=libsdgr_bg.so SDGR_EXTRA_FLAGS=-DSDGR_BIG_WALK_PAIRS=2000000000 SDGR_BUILD_SUFFIX=_bg python paper_2506_21633_b200/csrc/build.py
mkdir -p gpurun_out
for lib in libsdgr_sm.so libsdgr_bg.so; do
  SDGR_LIB=$lib timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/variant_$lib.log 2>&1
  echo "$lib rc=$?"; tail -2 gpurun_out/variant_$lib.log
done
