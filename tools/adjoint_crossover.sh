for c in 1024 2048 3072; do
  for v in lane cta; do
    echo -n "cands $c $v :: "
    DGX_ADJ=$v timeout 600 python bench.py --workload config3 --candidates $c --steps 6 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value']), {k:round(v['avg_launch_ms'],2) for k,v in d['roofline']['kernels'].items()})"
  done
done
