#!/bin/bash
# c3 (n = 16) on the single-pass orbit-pattern executor: tests, bench A/B against
# the two-pass executor, launch list and one ncu --set full capture.
set -u
O=gpurun_out/c3; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "n16 or alternative or real_io or scratch" > $O/gputest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/gputest.log
for ex in auto orbit-two-pass; do
  timeout 600 python bench.py --config c3 --executor $ex --no-cpu --no-e2e > $O/bench_c3_$ex.json 2> $O/bench_c3_$ex.err; echo "bench $ex rc=$?"
  python - $O/bench_c3_$ex.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d['roofline']; print(' ', d['value'], 'fwd', r['fwd_ms'], 'inv', r['inv_ms'], 'frac', r['frac'], 'rt', d.get('roundtrip_rel_err'))
PY
done
timeout 600 python bench.py --config c3 --real-io 0 --no-cpu --no-e2e > $O/bench_c3_complex.json 2> $O/bench_c3_complex.err; echo "bench complex rc=$?"; python -c "
import json;d=json.loads(open('$O/bench_c3_complex.json').read().strip().splitlines()[-1]);r=d['roofline'];print(' ',d['value'],'fwd',r['fwd_ms'],'inv',r['inv_ms'])"
if [ "${NCU:-1}" = 1 ]; then
timeout 900 ncu --set full --import-source on --clock-control none -k regex:orbit_pat -c 2 -o $O/orbit_pat_full -f python tools/prof_run.py --n 16 --blocks 16384 --real > $O/ncu.log 2>&1; echo "ncu rc=$?"
fi
