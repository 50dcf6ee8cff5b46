#!/bin/bash
# A/B timing on one box: alternate bench runs between two builds of
# libplaid.so (PLAID_LIB), so box-to-box variance cancels.
#   tools/ab.sh <libA.so> <libB.so> [rounds] [bench args...]
set -u
a=$1; b=$2; n=${3:-3}; shift 3 || shift $#
for i in $(seq "$n"); do
    for lib in "$a" "$b"; do
        PLAID_LIB=$lib python bench.py --steps 400 --warmup 20 --no-cpu "$@" 2>/dev/null | tail -1 |
            python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $lib)', round(d['value'],1), round(d['p50_ms']*1e3,1), round(d['e2e']['value'],1))"
    done
done
