#!/bin/bash
# Round-2 verification pass on one B200: GPU tests, smoke, every config's bench line.
# Output under gpurun_out/r02v/ (copied to profiles/ by hand after review).
set -u
O=gpurun_out/r02v; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/gputest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
run() {  # tag, args...
  local tag=$1; shift
  timeout 600 python bench.py "$@" > $O/bench_$tag.json 2> $O/bench_$tag.err
  echo "bench $tag rc=$?"
  python - "$O/bench_$tag.json" <<'PY' || tail -5 $O/bench_$tag.err
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}; c=d.get('cpu_baseline') or {}; e=d.get('e2e') or {}
print(' ', d['value'], d['unit'], 'fwd', r.get('fwd_ms'), 'inv', r.get('inv_ms'), 'frac', r.get('frac'), 'rt', d.get('roundtrip_rel_err'), 'cpu', c.get('value'), 'e2e', e.get('value'))
PY
}
run c2 ${BENCH_ARGS:-}
run c1 --config c1
run c3 --config c3
run c3d --config c3 --method direct --blocks 1024
run c4 --config c4
run c5 --config c5
run c2f32 --precision f32 --no-cpu
run c2d --method direct
run c2f32d --method direct --precision f32 --no-cpu
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "reference rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1; echo "ncu launches rc=$?"
# c3's dominant kernel: one ncu --set full capture (forward + inverse launch) and the raw page
timeout 900 ncu --set full --import-source on --clock-control none -k regex:orbit_pat_kernel -c 2 -o $O/orbit_pat_full -f python tools/prof_run.py --n 16 --blocks 16384 --real > $O/ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv python bench.py --config c3 --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1; echo "ncu launches c3 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv python bench.py --config c4 --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1; echo "ncu launches c4 rc=$?"
