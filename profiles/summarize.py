"""Summaries committed under profiles/ from ncu captures brought back by gpurun.

  python profiles/summarize.py full REPORT.ncu-rep OUT.json     # one entry per kernel launch (--set full)
  python profiles/summarize.py launches LAUNCHES.csv OUT.csv    # gpu__time_duration.sum launch list -> per-kernel shares
  python profiles/summarize.py traffic SUMMARY.json OUT.json     # blend launch's DRAM bytes -> bench.py roofline.traffic

The launch list is cold-cache and serialised (ncu replays each launch alone), so only
each kernel's SHARE of the frame is comparable with bench.py, not the absolute time.
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
]


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        e = {"kernel": d.get("Kernel Name", "")[:160], "id": d.get("ID")}
        for k in KEYS:
            if k in d:
                try:
                    e[k] = [float(d[k].replace(",", "")), u.get(k, "")]
                except ValueError:
                    e[k] = [d[k], u.get(k, "")]
        st = {k[len("smsp__pcsamp_warps_issue_stalled_"):]: float(d[k].replace(",", "") or 0) for k in hdr
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
        tot = sum(st.values()) or 1.0
        e["stall_top_pct"] = {k: round(v / tot * 100, 1) for k, v in sorted(st.items(), key=lambda t: -t[1])[:8]}
        res.append(e)
    json.dump(res, open(out, "w"), indent=1)
    print(f"{out}: {len(res)} launches")


def launches(csv_in, out):
    lines = [l for l in open(csv_in) if not l.startswith("==")]
    rows = list(csv.reader(lines))
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    rows = [r for r in rows[1:] if len(r) > vi]
    starts = [i for i, r in enumerate(rows) if "frame_init_kernel" in r[ki]]
    if not starts:  # captures before the one-kernel frame reset started at preprocess
        starts = [i for i, r in enumerate(rows) if "preprocess_kernel" in r[ki]]
    if starts:  # keep the last frame (from its first launch; memsets are not kernels)
        s0 = starts[-1]
        if s0 > 0 and "assign_labels" in rows[s0 - 1][ki]:  # render_panoptic frames start at assign_labels
            s0 -= 1
        rows = rows[s0:]
    agg = {}
    for r in rows:
        name = r[ki].split("(")[0].replace("void ", "").replace("psm::<unnamed>::", "")
        v = float(r[vi].replace(",", ""))
        v = v / 1000.0 if r[ui] in ("ns", "nsecond") else (v * 1000.0 if r[ui] in ("ms", "msecond") else v)
        agg.setdefault(name, []).append(v)
    tot = sum(sum(v) for v in agg.values())
    with open(out, "w") as f:
        f.write("kernel,launches,time_us_total,share\n")
        for k, v in sorted(agg.items(), key=lambda t: -sum(t[1])):
            f.write(f"\"{k}\",{len(v)},{sum(v):.1f},{sum(v) / tot:.3f}\n")
    print(f"{out}: {len(agg)} kernels, {tot:.1f} us")


def traffic(summary_json, out):
    """The last blend_kernel launch of a `full` summary (one frame's K7) -> the per-launch DRAM
    traffic that bench.py reports as roofline.traffic."""
    ents = [e for e in json.load(open(summary_json)) if e["kernel"].startswith(("blend_kernel", "void psm::blend"))
            or "blend_kernel" in e["kernel"]]
    if not ents:
        raise SystemExit("no blend_kernel launch in " + summary_json)
    e = ents[-1]
    rd, wr = e["dram__bytes_read.sum"][0], e["dram__bytes_write.sum"][0]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd *= scale.get(e["dram__bytes_read.sum"][1], 1)
    wr *= scale.get(e["dram__bytes_write.sum"][1], 1)
    json.dump({"kernel": e["kernel"], "source": summary_json + " (ncu --set full --clock-control none, "
               "python profiles/frame.py c3 2; profiles/capture.sh)", "dram_bytes_read": rd, "dram_bytes_write": wr,
               "dram_bytes_per_launch": rd + wr, "launch_us": e["gpu__time_duration.sum"]}, open(out, "w"), indent=1)
    print(f"{out}: {rd + wr:.0f} B per launch")


if __name__ == "__main__":
    {"full": full, "launches": launches, "traffic": traffic}[sys.argv[1]](sys.argv[2], sys.argv[3])
