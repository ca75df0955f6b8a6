"""Per-opcode shared-memory wavefronts (measured vs ideal) and the MIO slot share of a kernel from
an ncu --set full capture: python tools/ncu_wavefronts.py src.csv raw.csv
(src.csv: ncu -i rep --page source --csv --print-source sass; raw.csv: --page raw --csv)."""
import collections
import csv
import sys


def main(src, raw):
    rows = list(csv.reader(open(src)))
    hi = [i for i, r in enumerate(rows) if 'Address' in r and 'Source' in r][0]
    h = rows[hi]
    ix = {k: i for i, k in enumerate(h)}
    seen, data = set(), []
    for r in rows[hi + 1:]:
        if r[ix['Address']] not in seen:
            seen.add(r[ix['Address']])
            data.append(r)

    def f(r, k):
        try:
            return float(r[ix[k]].replace(',', ''))
        except (ValueError, KeyError):
            return 0.0
    wf, ideal, ins, n = (collections.Counter() for _ in range(4))
    shfl = 0.0
    for r in data:
        src_ = r[ix['Source']].strip()
        op = src_.split()[1] if src_.startswith('@') else (src_.split() or [''])[0]
        if op.startswith('SHFL'):
            shfl += f(r, 'Instructions Executed')
        w = f(r, 'L1 Wavefronts Shared')
        if w > 0:
            wf[op] += w
            ideal[op] += f(r, 'L1 Wavefronts Shared Ideal')
            ins[op] += f(r, 'Instructions Executed')
            n[op] += 1
    print(f"{'opcode':10s} {'static':>6s} {'executed':>12s} {'wavefronts':>12s} {'ideal':>12s} {'wf/instr':>8s}")
    for k, v in wf.most_common():
        print(f"{k:10s} {n[k]:6d} {ins[k]:12.4g} {v:12.4g} {ideal[k]:12.4g} {v / ins[k]:8.2f}")
    tw, ti = sum(wf.values()), sum(ideal.values())
    print(f"total wavefronts {tw:.4g} (ideal {ti:.4g}, excess {100 * (tw / ti - 1):.1f}%), SHFL {shfl:.4g}")
    r = list(csv.reader(open(raw)))
    d = dict(zip(r[0], r[2]))
    cyc = float(d['sm__cycles_elapsed.avg'].replace(',', ''))
    nsm = 148
    wf_all = float(d['l1tex__data_pipe_lsu_wavefronts_mem_shared.sum'].replace(',', ''))
    print(f"per SM: {wf_all / nsm:.4g} wavefronts + {shfl / nsm:.4g} shuffles over {cyc:.4g} cycles = "
          f"{100 * (wf_all + shfl) / nsm / cyc:.1f}% of one MIO slot per clock "
          f"(wavefronts alone {100 * wf_all / nsm / cyc:.1f}%)")


if __name__ == '__main__':
    main(sys.argv[1], sys.argv[2])
