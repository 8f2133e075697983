#!/bin/bash
# One gpurun call: selected parity tests + short bench (stage times).  usage: tools/ab.sh TAG "pytest -k expr" [extra bench args]
TAG=$1; K=${2:-"backward or full_step or graph or trained or dense"}; shift 2
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_scale_gpu.py ${EXTRA_TESTS} -x -q -k "$K" > gpurun_out/${TAG}_pytest.log 2>&1; tail -3 gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 5 --trained-steps 0 "$@" > gpurun_out/${TAG}_bench.jsonl 2>gpurun_out/${TAG}_bench.err
python -c "import json;d=json.load(open('gpurun_out/${TAG}_bench.jsonl'));print(round(d['value'],1), d['stages_ms'])" || tail -5 gpurun_out/${TAG}_bench.err
