"""Per-source-line instruction / stall-sample shares of one kernel in an ncu report
(python tools/ncu_lines.py REPORT KERNEL_REGEX [TOP] [LAUNCH_SKIP]); reads `ncu --page source --print-source cuda,sass`
(all matching launches, or only the one after LAUNCH_SKIP of them)."""
import csv, io, subprocess, sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
skip = ["--launch-skip", sys.argv[4], "--launch-count", "1"] if len(sys.argv) > 4 else []
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kre]
                     + skip, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
lines, cur, fname = {}, None, ""
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        if r[0] == "Line No":
            hdr = r
            ie, sm = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if r[0]:
        cur = (fname, r[0], r[1].strip()[:90])
        lines.setdefault(cur, [0, 0])
    elif cur is not None:
        try:
            lines[cur][0] += int(r[ie]); lines[cur][1] += int(r[sm])
        except (ValueError, IndexError):
            pass
ti = sum(v[0] for v in lines.values()) or 1
ts = sum(v[1] for v in lines.values()) or 1
print(f"total inst {ti/1e6:.2f}M samples {ts}")
for k, v in sorted(lines.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{v[0]/ti*100:5.1f}% inst {v[1]/ts*100:5.1f}% smp  {k[0]}:{k[1]}  {k[2]}")
