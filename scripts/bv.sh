# usage: bv.sh label [env...] -- bench cfg3 600 steps, print value
label=$1; shift
env "$@" python bench.py --steps 600 --warmup 12 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$label', round(d['value'],1), d['clocks']['sm_mhz'], d['max_abs_trace_err'])"
