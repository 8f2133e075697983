#!/bin/bash
# quick GPU check: selected parity tests + a short bench with per-stage times.  usage: tools/quick.sh TAG "pytest -k expr"
TAG=$1; K=${2:-"loss or full_step or graph or sharded"}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "$K" > gpurun_out/${TAG}_pytest.log 2>&1; tail -3 gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --e2e-steps 5 > gpurun_out/${TAG}_bench.jsonl 2>gpurun_out/${TAG}_bench.err
python -c "import json;d=json.load(open('gpurun_out/${TAG}_bench.jsonl'));print(round(d['value'],1), d['stages_ms'])" || tail -5 gpurun_out/${TAG}_bench.err
