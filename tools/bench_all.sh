#!/bin/bash
# Every BASELINE config through bench.py, one JSON line each -> gpurun_out/bench_r02_configs.jsonl
# usage (on the GPU box): tools/bench_all.sh [extra bench.py args]
out=gpurun_out/bench_r02_configs.jsonl
mkdir -p gpurun_out; : > $out
run() { echo "== $*" >&2; timeout 900 python bench.py --steps 5 --warmup 3 "$@" >> $out 2>> gpurun_out/bench_all.err || echo "{\"failed\": \"$*\"}" >> $out; }
run --config 3 "$@"
run --config 0 "$@"
run --config 1 --case m2m "$@"
run --config 1 --case l2l "$@"
run --config 2 "$@"
run --config 4 --case 24to12 "$@"
run --config 4 --case 12to24 "$@"
for p in 2 4 6 8 10 12 14 16 18 20 21 22 24 26 28 30; do run --config 4 --case p$p "$@"; done
cat $out | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l)
    if 'failed' in d: print(d); continue
    r = d['roofline']
    print('%-60s %10.3e tr/s  %8.3f ms  %s frac=%.3f  e2e=%.3e  cpu=%.3e' % (d['config']['workload'][:60], d['value'], d['ms_per_step'], r['bound'], r['frac'], d.get('e2e', {}).get('value', float('nan')), d.get('cpu_baseline', {}).get('value', float('nan'))))
"
