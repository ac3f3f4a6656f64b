#!/bin/bash
# One GPU session: bench line, ncu launch list, ncu --set full of k_fused3 launches (TMA-staged
# ring slot p0 = 3, plain-load slots p0 = 12 and 0), GPU tests.  Outputs under gpurun_out/.
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 60 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
# perp.py launch order: p0 = 0, 3, 6, 9, 12, 1, ... (groups of 3 from k = L = 14)
for sk in 1 4 0; do
  ncu --set full --clock-control none --import-source on -k regex:k_fused3 -s $sk -c 1 -o gpurun_out/prof_s$sk -f \
      python scripts/perp.py --reps 0 > gpurun_out/ncu_s$sk.log 2>&1
  python scripts/ncu_summary.py gpurun_out/prof_s$sk.ncu-rep gpurun_out/prof_s$sk.json > /dev/null
  [ $sk != 1 ] && rm -f gpurun_out/prof_s$sk.ncu-rep   # keep one report (gpurun copies back <= 64 MiB)
done
python scripts/perp.py > gpurun_out/perp.txt 2>&1
timeout 1800 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
ls -la gpurun_out; du -sh gpurun_out
