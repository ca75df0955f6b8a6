"""Summarise an ncu --set full capture of k_fit: key counters, stall reasons, hot-loop SASS mix.
usage: python tools/ncu_summary.py raw.csv src.csv"""
import collections
import csv
import sys

KEYS = ['gpu__time_duration.sum', 'launch__registers_per_thread', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'lts__t_bytes.sum']
STALLS = ['short_scoreboard', 'wait', 'long_scoreboard', 'math_pipe_throttle', 'not_selected', 'mio_throttle',
          'dispatch_stall', 'branch_resolving', 'no_instruction', 'lg_throttle', 'barrier', 'membar']


def main(raw, src):
    r = list(csv.reader(open(raw)))
    d = dict(zip(r[0], r[2]))
    for k in KEYS:
        if k in d:
            print(f"{k:80s} {d[k]} {r[1][r[0].index(k)]}")
    for s in STALLS:
        k = f'smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio'
        if k in d:
            print(f"stall {s:22s} {float(d[k]):.3f}")
    rows = list(csv.reader(open(src)))
    h = rows[1]
    ix = {k: i for i, k in enumerate(h)}
    data = rows[2:]

    def f(row, k):
        try:
            return float(row[ix[k]].replace(',', ''))
        except (ValueError, KeyError):
            return 0.0
    mx = max(f(x, 'Instructions Executed') for x in data)
    hot = [x for x in data if f(x, 'Instructions Executed') > 0.5 * mx]
    ops = collections.Counter((x[ix['Source']].split()[1] if x[ix['Source']].strip().startswith('@')
                               else x[ix['Source']].split()[0]) for x in hot)
    print(f"hot loop: {len(hot)} static instrs executed ~{mx:.3g} times; mix:",
          ", ".join(f"{k} {v}" for k, v in ops.most_common()))


if __name__ == '__main__':
    main(sys.argv[1], sys.argv[2])
