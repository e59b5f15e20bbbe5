#!/bin/bash
# per-stage clock breakdown under env-switched variants
for v in "$@"; do echo "== $v"; env $v python tools/stage_timing.py 8 2>&1 | head -1; done
