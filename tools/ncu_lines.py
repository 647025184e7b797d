"""Per-source-line instruction / stall-sample shares of one kernel in an ncu
--set full capture (needs -lineinfo + --import-source on).

  python tools/ncu_lines.py rep.ncu-rep 'k_stream_grp<(int)1, (int)8>' [N]
"""
import csv
import io
import subprocess
import sys


def main(rep, pat, n=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur = h = kern = None
    res = []
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] in ("Kernel Name", "Function Name"):
            kern = r[1]
            continue
        if r[0] == "File Path":
            cur = r[1]
            continue
        if r[0] == "Line No":
            h = r
            continue
        if h and len(r) >= 8 and r[0] and kern and pat in kern:
            try:
                res.append((cur.split('/')[-1], int(r[0]), float(r[4] or 0), float(r[7] or 0), r[1][:100]))
            except ValueError:
                pass
    ts = sum(x[2] for x in res) or 1
    ti = sum(x[3] for x in res) or 1
    print(f"# {pat}: {ti:.0f} warp instructions, {ts:.0f} stall samples")
    for f, ln, s, i, src in sorted(res, key=lambda x: -x[3])[:n]:
        print(f"{f[:16]:16s}{ln:5d} inst {i / ti * 100:5.1f}% samp {s / ts * 100:5.1f}%  {src}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
