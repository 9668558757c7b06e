#!/usr/bin/env python
"""Summarise an ncu report (--set full): per kernel launch, the numbers the roofline and the
optimisation loop use.  Usage: python tools/ncu_summary.py report.ncu-rep [--out file.txt] [--json traffic.json]"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    ("time_us", "gpu__time_duration.sum", "us"),
    ("dram_rd_GB", "dram__bytes_read.sum", "GB"),
    ("dram_wr_GB", "dram__bytes_write.sum", "GB"),
    ("dram_%", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("l2_hit_%", "lts__t_sector_hit_rate.pct", 1),
    ("occ_%", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("regs", "launch__registers_per_thread", 1),
    ("issue_%", "sm__inst_issued.avg.pct_of_peak_sustained_active", 1),
    ("xu_%", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 1),
    ("lsu_%", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", 1),
    ("l1_wf_%", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", 1),
    ("lts_%", "lts__t_sectors.avg.pct_of_peak_sustained_elapsed", 1),
]
STALLS = ["long_scoreboard", "short_scoreboard", "lg_throttle", "mio_throttle", "wait", "math_pipe_throttle",
          "barrier", "membar", "no_instruction", "not_selected", "selected", "dispatch_stall", "tex_throttle",
          "drain", "branch_resolving", "sleeping"]


SCALE = {("us", "ns"): 1e-3, ("us", "us"): 1.0, ("us", "ms"): 1e3, ("us", "s"): 1e6,
         ("GB", "byte"): 1e-9, ("GB", "Kbyte"): 1e-6, ("GB", "Mbyte"): 1e-3, ("GB", "Gbyte"): 1.0,
         ("GB", "Tbyte"): 1e3}


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def from_text(path):
    """(header, units, rows) rebuilt from a saved summary text (its first three metric columns)."""
    h, units, rows = ["Kernel Name"], [""], []
    for n, m, _ in METRICS:
        h.append(m)
        units.append("")
    for line in open(path):
        parts = line.split()
        if not parts or parts[0] in ("kernel", "#", "stalls(cycles/issue):") or line.startswith(" "):
            continue
        # the name may contain spaces ("k_pool_fwd_f32<8, 2, 0, 1, 0, 1>"): numbers are the tail
        nums = parts[-len(METRICS):]
        name = line[:38].strip()
        rows.append([name] + nums)
    return h, units, rows


def main():
    rep = sys.argv[1]
    h, units, rows = from_text(rep) if rep.endswith(".txt") else load(rep)
    ki = h.index("Kernel Name")
    lines, traffic = [], {}
    hdr = f"{'kernel':38s} " + " ".join(f"{n:>10s}" for n, _, _ in METRICS)
    lines.append(hdr)
    for r in rows:
        name = r[ki].split("(")[0].replace("void ", "").replace("lirank::", "")[:38]
        vals = []
        for n, m, sc in METRICS:
            try:
                i = h.index(m)
                f = SCALE.get((sc, units[i]), 1.0) if isinstance(sc, str) else sc
                vals.append(float(r[i].replace(",", "")) * f)
            except (ValueError, IndexError):
                vals.append(float("nan"))
        lines.append(f"{name:38s} " + " ".join(f"{v:10.3f}" for v in vals))
        st = []
        for s in STALLS:
            m = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if m in h:
                try:
                    v = float(r[h.index(m)].replace(",", ""))
                    if v > 0.5:
                        st.append(f"{s}={v:.1f}")
                except ValueError:
                    pass
        if st:
            lines.append(f"{'':38s}   stalls(cycles/issue): " + " ".join(st))
        rd = vals[1] + vals[2]
        traffic.setdefault(name, []).append(rd * 1e9)  # per instantiation (template arguments kept)
    text = "\n".join(lines)
    print(text)
    if "--out" in sys.argv:
        open(sys.argv[sys.argv.index("--out") + 1], "w").write(f"# ncu summary of {rep}\n" + text + "\n")
    if "--json" in sys.argv:
        # per library phase (emb_profile's phases; what bench.py's roofline.traffic reads): the
        # DRAM bytes of one instance of the phase = sum over its kernels of (bytes per launch x
        # launches per step); the capture is one step of tools/profile_step.py
        phases = {"fwd": ["k_pool_fwd_f32", "k_pool_short_f32", "k_len_hist", "k_len_scatter"],
                  "fwd_q8": ["k_pool_fwd_q8"], "sort": ["k_radix_hist", "k_hist_excl", "k_onesweep"],
                  "rle": ["k_rle"], "segreduce": ["k_segreduce", "k_fixup_short", "k_fixup_long", "k_fixup_long_pieces", "k_fixup_long_combine"],
                  "norm": ["k_norm_partial", "k_norm_finalize"], "update": ["k_adagrad_tma", "k_adagrad"],
                  "quantize": ["k_quantize"]}
        per_step = {"k_onesweep": 3}  # digit passes per step (27-bit Feed-1 keys)
        j = {"_source": f"ncu --set full --clock-control none, one step of tools/profile_step.py ({rep}); "
                        "dram__bytes_read.sum + dram__bytes_write.sum per phase instance"}
        # each distinct instantiation of a phase's kernels runs once per step (the sort's digit
        # passes: per_step times), e.g. a6's ALU-widening pass and its Inf/NaN re-run are summed
        for ph, ks in phases.items():
            tot, have = 0.0, []
            for name, v in traffic.items():
                base = name.split("<")[0]
                if base in ks:
                    tot += sum(v) / len(v) * per_step.get(base, 1)
                    have.append(name)
            if have:
                j[ph] = {"dram_bytes_per_launch": tot, "kernels": have}
        # phases this capture does not cover (e.g. the full-table a9) keep their earlier entries
        path = sys.argv[sys.argv.index("--json") + 1]
        try:
            old = json.load(open(path))
            for ph, v in old.items():
                if ph not in j and not ph.startswith("_"):
                    j[ph] = dict(v, note=v.get("note", "from an earlier capture: " + old.get("_source", "")[-60:]))
        except (OSError, ValueError):
            pass
        json.dump(j, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
