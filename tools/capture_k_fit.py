"""ncu capture of the shipped k_fit launch that bench.py times (run on the GPU box, 1 GPU):

  python tools/capture_k_fit.py run     # plain bench run, then the same command under ncu
  python tools/capture_k_fit.py parse gpurun_out/k_fit_metrics.csv   # -> profiles/r02_k_fit_capture.json

The JSON is keyed by the hash of the kernel sources (bench.source_hash) and the launch
(windows, events, evaluations): bench.py reports its `traffic` (DRAM bytes) and the measured
MIO occupancy only when both match, so a number is never carried over to a different kernel."""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

CMD = ["python", "bench.py", "--no-sub", "--no-e2e", "--no-cpu", "--steps", "1", "--warmup", "1"]
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__cycles_elapsed.avg", "smsp__inst_executed.sum",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
           "l1tex__data_pipe_lsu_wavefronts.sum", "l1tex__data_pipe_lsu_wavefronts_mem_lg.sum"]
OUT = os.path.join(ROOT, "gpurun_out", "k_fit_metrics.csv")


def run():
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    r = subprocess.run(CMD, cwd=ROOT, capture_output=True, text=True)
    line = r.stdout.strip().splitlines()[-1]
    open(os.path.join(ROOT, "gpurun_out", "k_fit_capture_plain.jsonl"), "w").write(line + "\n")
    if r.returncode != 0:
        print(r.stderr[-2000:])
        return r.returncode
    # the second k_fit launch is the timed step of CMD (the first is the warm-up)
    ncu = ["ncu", "--metrics", ",".join(METRICS), "--clock-control", "none", "-k", "regex:k_fit", "-s", "1",
           "-c", "1", "--csv", "--log-file", OUT] + CMD
    r2 = subprocess.run(ncu, cwd=ROOT, capture_output=True, text=True)
    print(r2.stdout[-1500:], r2.stderr[-1500:])
    return r2.returncode


def parse(path):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    vals, units = {}, {}
    for r in rows[1:]:
        if len(r) < len(h) or "k_fit" not in r[ix["Kernel Name"]]:
            continue
        name = r[ix["Metric Name"]]
        try:
            vals[name] = float(r[ix["Metric Value"]].replace(",", ""))
        except ValueError:   # "n/a": not collectable on this driver
            continue
        units[name] = r[ix["Metric Unit"]]
        kernel = r[ix["Kernel Name"]]
    plain = json.loads(open(os.path.join(ROOT, "gpurun_out", "k_fit_capture_plain.jsonl")).read())
    cfgj = plain["config"]
    W, E = cfgj["windows"], cfgj["per_rank"]["events"][0]
    evals = cfgj["iterations"] + 1
    ev_eval = cfgj["event_evaluations_per_step"]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "B": 1, "KB": 1e3, "MB": 1e6,
             "GB": 1e9, "TB": 1e12}
    b = lambda k: vals[k] * scale.get(units[k], 1.0)
    dram = b("dram__bytes_read.sum") + b("dram__bytes_write.sum")
    lts = b("lts__t_bytes.sum")
    wf = vals["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
    cyc = vals["sm__cycles_elapsed.avg"]
    # warp shuffles share the MIO slot with shared wavefronts (profiles/r01_ubench_b200.txt); the
    # op_shfl counter is not collectable on this driver, so the SASS count per event is used
    shfl_per_ev = 9 / 16
    mio = (wf + shfl_per_ev * ev_eval) / (148 * cyc)
    out = {"kernel": kernel.split("(")[0], "source_hash": bench.source_hash(), "windows": W, "events": E,
           "evaluations": evals, "event_evaluations": ev_eval, "gpu_time_s": vals["gpu__time_duration.sum"] * {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6,
                                                            "ms": 1e-3, "msecond": 1e-3}[units["gpu__time_duration.sum"]],
           "dram_bytes": dram, "dram_bytes_per_event_evaluation": dram / ev_eval, "l2_bytes": lts,
           "shared_wavefronts": wf, "shared_wavefronts_per_event_evaluation": wf / ev_eval,
           "bank_conflicts": vals.get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
           "sm_cycles": cyc, "mio_frac": mio,
           "mio_basis": f"(shared wavefronts + {shfl_per_ev:.4f} SHFL per event-evaluation from the SASS) / (148 SMs x cycles)",
           "issue_active_pct": vals.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
           "mufu_pct": vals.get("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
           "inst_executed": vals.get("smsp__inst_executed.sum"),
           "global_ld_sectors": vals.get("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"),
           "lsu_wavefronts_all": vals.get("l1tex__data_pipe_lsu_wavefronts.sum"),
           "lsu_wavefronts_global": vals.get("l1tex__data_pipe_lsu_wavefronts_mem_lg.sum"),
           "mio_frac_incl_global": ((vals["l1tex__data_pipe_lsu_wavefronts.sum"] + shfl_per_ev * ev_eval) / (148 * cyc)
                                    if "l1tex__data_pipe_lsu_wavefronts.sum" in vals else None),
           "command": " ".join(CMD), "metrics_csv": os.path.relpath(path, ROOT)}
    dst = os.path.join(ROOT, "profiles", "r02_k_fit_capture.json")
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        sys.exit(run())
    parse(sys.argv[2] if len(sys.argv) > 2 else OUT)
