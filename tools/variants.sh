#!/bin/bash
# A/B the HS_FFT_VARIANT plans: parity of the planned grids + a short bench per variant.
for v in ${VARIANTS:-0 1 2 3}; do
  export HS_FFT_VARIANT=$v
  r=$(timeout 300 python -m pytest tests/test_parity_gpu.py -x -q -k "static_plans or cfg2_grid" 2>&1 | tail -1)
  b=$(timeout 300 python bench.py --steps 150 --warmup 5 --no-cpu-baseline --e2e-steps 5 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());s=d['stages_ms'];print(round(d['value'],1),{k:s[k] for k in ('rows_fwd','cols_fwd','rows_inv','rows_fwd_bwd','cols_bwd','rows_inv_bwd')})")
  echo "variant $v: $r | $b"
done
