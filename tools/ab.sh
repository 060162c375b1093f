#!/bin/bash
# A/B timing of alternative library builds on the same box: tools/ab.sh "ENV=.. ENV2=.." lib1.so lib2.so ...
# (each line: library, env, config-1 call times, it/s; config 3)
envs="$1"; shift
for rep in 1 2; do
for lib in "$@"; do
  env $envs LX_LIBRARY=$lib timeout 300 python tools/sweep.py --only 1,3 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print('$lib'.split('/')[-1], d['config'], [round(c['ms'],4) for c in d['calls']], round(d['leja_it_per_s']))
"
done
done
