#!/bin/bash
# compare fusion depths / kernel variants on the bench workload (short runs, no cpu baseline / e2e)
for cfg in ${CFGS:-"1 warp" "2 warp" "2 reg"}; do
  set -- $cfg
  echo -n "fuse $1 kind $2: "
  QUAPI_FUSE_S=$1 QUAPI_FUSED_KIND=$2 python bench.py --steps ${STEPS:-1000} --warmup 10 --no-cpu-baseline --no-e2e ${EXTRA} | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],4), round(d['roofline']['achieved']), round(d['roofline']['frac'],3), d['gpu_launches'], d['config']['grid'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
