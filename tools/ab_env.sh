#!/bin/bash
# A/B an env knob: tools/ab_env.sh VAR "v1 v2 ..." [pytest -k expr]
VAR=$1; VALS=$2; K=${3:-"loss or full_step"}
for v in $VALS; do
  export $VAR=$v
  r=$(timeout 300 python -m pytest tests/test_parity_gpu.py -x -q -k "$K" 2>&1 | tail -1)
  b=$(timeout 300 python bench.py --steps 150 --warmup 5 --no-cpu-baseline --e2e-steps 5 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],1),d['stages_ms'])")
  echo "$VAR=$v: $r | $b"
done
