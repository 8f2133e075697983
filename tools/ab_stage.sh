#!/bin/bash
# Stage times only (no parity) of builds build_ab/NAME.so: usage tools/ab_stage.sh "a b"
for n in $1; do
  export HOLOSPLAT_LIB=$PWD/build_ab/$n.so
  b=$(timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 3 --trained-steps 0 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],1),{k:round(v*1e3,1) for k,v in d['stages_ms'].items()})")
  echo "$n: $b"
done
