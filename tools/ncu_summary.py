"""Compact summary of an `ncu --set full` capture (.ncu-rep) for profiles/.

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/rNN_<kernel>.txt

Prints, per captured launch, the metrics the roofline discussion cites
(duration, DRAM bytes, DRAM / SM throughput, occupancy, registers, cache hit
rates) and the ncu rule findings with their estimated speed-ups.
"""
import csv
import io
import subprocess
import sys

RAW = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn_smem"),
    ("lts__t_sector_hit_rate.pct", "L2_hit_%"),
    ("l1tex__t_sector_hit_rate.pct", "L1_hit_%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_%"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu_pipe_%"),
    ("smsp__inst_executed.sum", "inst_executed"),
]


def ncu(path, page):
    out = subprocess.run(["ncu", "-i", path, "--page", page, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(path):
    rows = ncu(path, "raw")
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full summary of {path.split('/')[-1]}")
    for r in rows[2:]:
        print(f"\n## launch {r[hdr.index('ID')]}: {r[hdr.index('Kernel Name')]}")
        for key, label in RAW:
            if key in hdr:
                i = hdr.index(key)
                print(f"  {label:16s} {r[i]:>14s} {units[i]}")
        scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
        try:
            ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
            mb = float(r[ir]) * scale[units[ir]] + float(r[iw]) * scale[units[iw]]
            print(f"  {'traffic':16s} {mb:14.3f} Mbyte (read+write)")
        except (ValueError, KeyError):
            pass
    det = ncu(path, "details")
    h = det[0]
    seen = set()
    print("\n## ncu rule findings (first launch)")
    for r in det[1:]:
        if len(r) < len(h):
            continue
        rule, desc, sp = r[h.index("Rule Name")], r[h.index("Rule Description")], r[h.index("Estimated Speedup")]
        if rule and rule not in seen and r[h.index("ID")] == det[1][h.index("ID")]:
            seen.add(rule)
            print(f"- [{rule}] (est. speedup {sp or '-'}%) {desc[:400]}")


if __name__ == "__main__":
    main(sys.argv[1])
