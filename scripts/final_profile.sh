#!/bin/bash
# End-of-round GPU session: sanitizers, bench line, launch list, ncu of the top kernel (summary + warp
# stalls, the .ncu-rep stays on the box), per-slot launch times, sweep / eta benchmarks, GPU tests.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  echo "== $tool"; timeout 900 compute-sanitizer --tool $tool python scripts/sanitize_run.py 2>&1 | grep -E "sanitize run ok|SUMMARY|Error|error" | head -5
done > gpurun_out/sanitize.txt 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 60 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python scripts/launches_json.py gpurun_out/launches.csv gpurun_out/launches.json > /dev/null
for sk in 1 4 0 9; do   # perp.py launch order: p0 = 0, 3, 6, 9, 12, 1, 4, 7, 10, 13, ...
  ncu --set full --clock-control none --import-source on -k regex:k_fused3 -s $sk -c 1 -o /tmp/prof_s$sk -f \
      python scripts/perp.py --reps 0 > /tmp/ncu_s$sk.log 2>&1
  python scripts/ncu_summary.py /tmp/prof_s$sk.ncu-rep gpurun_out/prof_s$sk.json > /dev/null
  python scripts/ncu_stalls.py /tmp/prof_s$sk.ncu-rep 8 > gpurun_out/stalls_s$sk.json
done
python scripts/perp.py > gpurun_out/perp.txt 2>&1
{ timeout 600 python scripts/sweep_bench.py --L 5; timeout 600 python scripts/sweep_bench.py --L 7;
  timeout 900 python scripts/sweep_bench.py --L 9 --no-cpu-baseline;
  timeout 600 python scripts/sweep_bench.py --L 5 --temperature-sweep; } > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
timeout 300 python scripts/eta_bench.py > gpurun_out/eta_bench.jsonl 2> gpurun_out/eta_bench.err
timeout 1800 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
tail -2 gpurun_out/pytest_gpu.txt; cat gpurun_out/sanitize.txt; tail -1 gpurun_out/perp.txt; du -sh gpurun_out
