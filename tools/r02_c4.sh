#!/bin/bash
# c4 (n = 64) with the S pass on the orbit-pattern tables: tests, bench A/B against
# the streamed / generated S pass, launch list.
set -u
O=gpurun_out/c4; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py -m gpu -q -x -k "large_n or scratch or determin or canar" > $O/gputest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/gputest.log
for ex in auto orbit-streamed; do
  timeout 600 python bench.py --config c4 --executor $ex --no-cpu --no-e2e > $O/bench_c4_$ex.json 2> $O/bench_c4_$ex.err; echo "bench $ex rc=$?"
  python - $O/bench_c4_$ex.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d['roofline']; print(' ', d['value'], 'fwd', r['fwd_ms'], 'inv', r['inv_ms'], 'frac', r['frac'], 'rt', d.get('roundtrip_rel_err'))
PY
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv python tools/prof_run.py --n 64 --blocks 1 --reps 3 > /dev/null 2>&1; echo "ncu rc=$?"
grep -v "^==" $O/launches_c4.csv | awk -F'","' 'NR>1{print $5, $NF}' | tail -12
