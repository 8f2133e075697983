#!/bin/bash
# A/B two builds of libholosplat.so on the GPU box: build_ab/*.so (made here with
# tools/ab_make.sh NAME) timed by the same bench in turn, plus the selected parity tests.
# usage (on the box): tools/ab_build.sh "base new" [pytest -k expr] [steps]
NAMES=$1; K=${2:-"loss or full_step or backward"}; STEPS=${3:-300}
for n in $NAMES; do
  export HOLOSPLAT_LIB=$PWD/build_ab/$n.so
  r=$(timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "$K" 2>&1 | tail -1)
  b=$(timeout 600 python bench.py --steps $STEPS --warmup 10 --no-cpu-baseline --e2e-steps 5 --trained-steps 0 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],1),{k:round(v*1e3,1) for k,v in d['stages_ms'].items()})")
  echo "$n: $r | $b"
done
