"""Summaries of ncu captures for profiles/ (run here, no GPU needed).

python tools/ncu_summary.py launches <launches.csv>           -> per-kernel time shares
python tools/ncu_summary.py full <report.ncu-rep> [--json out] -> key metrics of the capture
"""
import collections
import csv
import json
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if len(r) > 5 and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                unit = d.get("Metric Unit", "ns")
                v = float(d["Metric Value"].replace(",", ""))
                v *= {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
                agg[d["Kernel Name"]][0] += 1
                agg[d["Kernel Name"]][1] += v
    tot = sum(v[1] for v in agg.values())
    out = []
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append({"kernel": k[:160], "launches": n, "total_us": t / 1e3, "share": t / tot, "avg_us": t / n / 1e3})
    return out


KEYS = ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread", "launch__block_size",
        "launch__grid_size", "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", "sm__cycles_elapsed.avg.per_second"]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (v, u) for h, v, u in zip(hdr, vals, units)}
    res = {"kernel": d.get("Kernel Name", ("", ""))[0][:160]}
    for k in KEYS:
        if k in d:
            res[k] = d[k][0] + (" " + d[k][1] if d[k][1] else "")
    st = {k: float(v[0]) for k, v in d.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")
          and v[0].replace(".", "").isdigit()}
    tot = sum(st.values()) or 1
    res["stall_shares"] = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): round(v / tot, 3)
                           for k, v in sorted(st.items(), key=lambda x: -x[1])[:10]}
    return res


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    res = launches(path) if mode == "launches" else full(path)
    txt = json.dumps(res, indent=1)
    if "--json" in sys.argv:
        open(sys.argv[sys.argv.index("--json") + 1], "w").write(txt + "\n")
    print(txt)
