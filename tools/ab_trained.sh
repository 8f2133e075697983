for n in $1; do
  export HOLOSPLAT_LIB=$PWD/build_ab/$n.so
  r=$(timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_parity_scale_gpu.py -x -q -k "backward or saturation or tails or trained or dense or cfg2_full" 2>&1 | tail -1)
  b=$(timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 5 --trained-steps 1000 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],1), 'trained', round(d['trained']['value'],1), 'bwd', d['stages_ms']['raster_bwd'])")
  echo "$n: $r | $b"
done
