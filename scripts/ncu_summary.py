"""Summarise an ncu --set full report (raw CSV page) for the kernels in it."""
import csv
import json
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread', 'launch__grid_size',
        'launch__block_size', 'launch__occupancy_limit_registers', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'lts__t_bytes.sum', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__cycles_elapsed.avg.per_second',
        'l1tex__t_sector_hit_rate.pct', 'lts__t_sector_hit_rate.pct',
        'smsp__average_warp_latency_issue_stalled_long_scoreboard', 'smsp__warps_issue_stalled_long_scoreboard_per_warp_active.pct',
        'smsp__warps_issue_stalled_lg_throttle_per_warp_active.pct', 'smsp__warps_issue_stalled_math_pipe_throttle_per_warp_active.pct',
        'smsp__warps_issue_stalled_wait_per_warp_active.pct', 'smsp__warps_issue_stalled_drain_per_warp_active.pct',
        'smsp__warps_issue_stalled_barrier_per_warp_active.pct', 'smsp__warps_issue_stalled_mio_throttle_per_warp_active.pct',
        'smsp__warps_issue_stalled_short_scoreboard_per_warp_active.pct', 'smsp__warps_issue_stalled_no_instruction_per_warp_active.pct',
        'smsp__warps_issue_stalled_not_selected_per_warp_active.pct', 'smsp__warps_issue_stalled_selected_per_warp_active.pct',
        'smsp__warps_issue_stalled_dispatch_stall_per_warp_active.pct', 'smsp__warps_issue_stalled_membar_per_warp_active.pct']


def main(rep, out_json=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    name_i = idx.get("Kernel Name")
    res = []
    for d in data:
        r = {"kernel": d[name_i] if name_i is not None else "?"}
        for w in WANT:
            if w in idx:
                v = d[idx[w]].replace(",", "")
                try:
                    r[w] = float(v)
                except ValueError:
                    r[w] = v
        res.append(r)
    for r in res:
        print(json.dumps(r))
    if out_json:
        with open(out_json, "w") as f:
            json.dump(res, f, indent=1)
    return res


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
