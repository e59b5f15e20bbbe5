set -x
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
tail -c 3000 gpurun_out/bench_c2.json
for args in "--n 16 --blocks 16384" "--n 16 --blocks 1024 --method direct" "--n 8 --precision f32" "--n 8 --method direct --precision f32" "--n 4 --blocks 262144" ; do
  python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e $args | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$args', d['value'], round(d['roofline']['fwd_ms'],4), round(d['roofline']['inv_ms'],4), round(d['roofline']['frac'],4), d['roundtrip_rel_err'])"
done
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/plain_bench.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1
python tools/prof_run.py > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:pipeline2 -c 2 -o gpurun_out/prof_r01_v2 python tools/prof_run.py > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
