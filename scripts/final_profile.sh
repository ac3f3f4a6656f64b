#!/bin/bash
# Round-end GPU profiling session (run from the repo root on a B200): bench lines of every config,
# the launch list of the default bench, ncu --set full of the top kernels (summaries + warp stalls;
# the .ncu-rep files come back in gpurun_out/), per-slot launch times.  The GPU test suite and
# smoke() run separately (scripts/final_checks.sh).
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
for c in 1 2 0 4 5; do
  timeout 900 python bench.py --cfg $c --no-cpu-baseline 2>> gpurun_out/bench_cfgs.err | tail -1
done > gpurun_out/bench_cfgs.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 60 --warmup 4 --reps 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python scripts/launches_json.py gpurun_out/launches.csv gpurun_out/launches.json > /dev/null
# k_fused4 on cfg3: two consecutive launches (two start slots) of the timed region
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused4 -s 6 -c 2 -o gpurun_out/prof_f4 -f \
    python bench.py --steps 40 --warmup 4 --reps 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_f4.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_f4.ncu-rep gpurun_out/prof_f4.json > /dev/null
python scripts/ncu_stalls.py gpurun_out/prof_f4.ncu-rep 8 > gpurun_out/stalls_f4.json
# k_fused2t on cfg4
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused2t -s 4 -c 2 -o gpurun_out/prof_f2t -f \
    python bench.py --cfg 4 --steps 20 --warmup 4 --reps 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_f2t.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_f2t.ncu-rep gpurun_out/prof_f2t.json > /dev/null
python scripts/ncu_stalls.py gpurun_out/prof_f2t.ncu-rep 8 > gpurun_out/stalls_f2t.json
timeout 300 python scripts/perp.py --cfg 4 > gpurun_out/perp4.txt 2>&1
timeout 300 python scripts/perp.py > gpurun_out/perp.txt 2>&1
timeout 300 python scripts/perp.py --final-only > gpurun_out/perp_final_only.txt 2>&1
tail -c 400 gpurun_out/bench.json; echo; cut -c1-200 gpurun_out/bench_cfgs.jsonl; tail -2 gpurun_out/perp.txt; du -sh gpurun_out
