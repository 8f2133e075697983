#!/bin/bash
# ncu --set full of selected kernels of an eager cfg2 step (1 GPU).  usage: tools/ncu_full.sh TAG REGEX [SKIP] [COUNT] [WORKLOAD]
TAG=$1; KRE=$2; SKIP=${3:-12}; CNT=${4:-6}; WL=${5:-cfg2}
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${KRE}" -s ${SKIP} -c ${CNT} \
   -o gpurun_out/${TAG}_full -f python tools/profile_step.py ${WL} 4 1 > gpurun_out/${TAG}_ncu.log 2>&1
tail -3 gpurun_out/${TAG}_ncu.log
