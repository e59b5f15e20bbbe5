#!/bin/bash
# A/B of env-switched kernel variants on the c2 bench (value = transforms/s)
for v in "$@"; do
  echo -n "$v: "
  env $v python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value']/1e6,2),'M/s fwd',round(r['fwd_ms'],4),'inv',round(r['inv_ms'],4),'frac',round(r['frac'],4))"
done
