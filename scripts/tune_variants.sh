#!/bin/bash
# sweep slide-kernel variants on the bench workload (short runs, no cpu baseline / e2e)
for v in ${VARIANTS:-3 5 6 7 8}; do
  echo -n "variant $v: "
  QUAPI_SLIDE_VARIANT=$v python bench.py --steps ${STEPS:-600} --warmup 10 --no-cpu-baseline --no-e2e ${EXTRA} | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'], d['config']['grid'], d['clocks']['sm_mhz'])"
done
