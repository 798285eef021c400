#!/bin/bash
# A/B of the cfg3 search launch on the GPU box: the library under tools/_bin/libgmpgr_base.so
# against the in-tree build, same workload, then the phase shares of the in-tree build.
#   tools/ab.sh [tag] [cfg] [kpxhops]
tag=${1:-ab}; cfg=${2:-cfg3}; kh=${3:--}
mkdir -p gpurun_out
if [ -f tools/_bin/libgmpgr_base.so ]; then
  GMPGR_LIB=tools/_bin/libgmpgr_base.so timeout 900 python tools/profile_search.py $cfg 65536 6 $kh tc > gpurun_out/${tag}_base.log 2>&1
fi
timeout 900 python tools/profile_search.py $cfg 65536 6 $kh tc > gpurun_out/${tag}_new.log 2>&1
GMPGR_PHASE_TIMING=1 timeout 900 python tools/profile_search.py $cfg 65536 3 $kh tc > gpurun_out/${tag}_phase.log 2>&1
tail -n 12 gpurun_out/${tag}_*.log
