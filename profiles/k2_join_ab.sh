#!/bin/bash
# Cost of joining K2 (LKV-H budgets, side stream) back into the eviction chain: default = K2
# signals the plan kernel through a workspace flag (K1 -> plan -> emit stay one PDL chain);
# LKV_K2_EVENT_JOIN = an event join before the plan; LKV_SERIAL_K2 = K2 before K1 on one stream.
cd "$(dirname "$0")/.."
t() { python bench.py --no-e2e --no-decode --no-cpu --steps 100 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readline()); print(round(d["ms_per_step"],4))'; }
for i in 1 2 3; do echo "flag $(t)"; echo "event_join $(LKV_K2_EVENT_JOIN=1 t)"; echo "serial $(LKV_SERIAL_K2=1 t)"; done
