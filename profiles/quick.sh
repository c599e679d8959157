#!/bin/bash
# quick GPU iteration: parity tests, then a short bench line
timeout -s KILL 900 python -m pytest tests -m gpu -x -q --timeout 600 2>&1 | tail -4
timeout -s KILL 300 python bench.py --no-e2e --no-cpu-baseline "$@" 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('ms/step %.2f  xterm %.2f ms  %.0f TOPS frac %.3f  phases %s key %s clocks %s' % (d['ms_per_step'], r['ms_per_launch'], r['achieved'], r['frac'], {k: round(v,3) for k,v in d['phases_ms_per_step'].items()}, d['key_recovered'], d.get('clocks')))"
