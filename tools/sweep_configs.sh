for c in c3 c4 c5; do
  python bench.py --config $c --steps 5 --warmup 3 --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$c.json').read()); print('$c', d['value'], d['unit'], round(d['roofline']['fwd_ms'],4), round(d['roofline']['inv_ms'],4), round(d['roofline']['frac'],4), d['roundtrip_rel_err'], (d['cpu_baseline'] or {}).get('value'))" || tail -5 gpurun_out/bench_$c.err
done
