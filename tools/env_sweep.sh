#!/bin/bash
# Bench the default workload under several engine env settings, one summary
# line per setting (ms_per_step, value, trace records, peak match).
#   tools/env_sweep.sh "MB_EVD_NE16=32" "MB_EVD_NE16=32 MB_EVD_NE32=64" ...
# The empty setting "" is the default configuration.
for setting in "$@"; do
  out=$(env $setting python bench.py --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1)
  echo "$out" | python -c "
import json, sys
d = json.loads(sys.stdin.read())
print(json.dumps({'env': '$setting', 'ms_per_step': round(d['ms_per_step'], 1), 'value': round(d['value'], 1),
                  'match': d['peak']['match'], 'p': d['peak']['probability'],
                  'records': d['contraction']['trace_records'], 'swaps': d['contraction']['accepted_swaps'],
                  'profile_ms': d.get('profile_ms')}))" || echo "{\"env\": \"$setting\", \"failed\": true}"
done
