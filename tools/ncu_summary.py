"""Summarise an ncu --set full report of the render kernel into markdown (for profiles/).

    python tools/ncu_summary.py REPORT.ncu-rep [--title T] > profiles/rNN_render_ncu.md
"""
import argparse
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads / warp instr"),
    ("sm__inst_executed.sum", "warp instructions"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/TEX throughput %"),
    ("l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed", "L1 data-pipe wavefronts %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 sector hit rate %"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "global load requests"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "global load sectors"),
    ("l1tex__t_sectors_pipe_tex_mem_texture.sum", "texture sectors"),
    ("l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", "local load sectors (stack pops)"),
    ("l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum", "local store sectors (stack pushes)"),
    ("l1tex__data_pipe_tex_wavefronts.sum.pct_of_peak_sustained_elapsed", "L1 texture data-pipe wavefronts %"),
    ("lts__t_sector_hit_rate.pct", "L2 sector hit rate %"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 read sectors (from L1)"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("dram__bytes_read.sum", "DRAM bytes read"),
    ("dram__bytes_write.sum", "DRAM bytes written"),
    ("dram__bytes.sum.per_second", "DRAM bandwidth"),
]


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--title", default="render_kernel")
    a = ap.parse_args()
    raw = ncu_csv(a.rep, "--page", "raw")
    h, units, vals = raw[0], raw[1], raw[2]
    idx = {n: i for i, n in enumerate(h)}
    print(f"# ncu summary: {a.title}\n")
    print(f"source: `{a.rep.split('/')[-1]}` (ncu --set full --clock-control none)\n")
    print("| metric | value | unit |\n|---|---|---|")
    for k, label in KEYS:
        if k in idx:
            print(f"| {label} (`{k}`) | {vals[idx[k]]} | {units[idx[k]]} |")
    # L2 read bandwidth actually served to L1 (sectors x 32 B / duration)
    dk, sk = "gpu__time_duration.sum", "lts__t_sectors_srcunit_tex_op_read.sum"
    if dk in idx and sk in idx:
        dur = float(vals[idx[dk]].replace(",", "")) * {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0}[units[idx[dk]]]
        gbs = float(vals[idx[sk]].replace(",", "")) * 32 / dur / 1e9
        print(f"| L2 -> L1 read bandwidth (`{sk}` x 32 B / duration) | {gbs:.1f} | GB/s |")
    # stall reasons
    sass = ncu_csv(a.rep, "--page", "source", "--print-source", "sass")
    sh = sass[1]
    si = {n: i for i, n in enumerate(sh)}
    rows = sass[2:]
    tot = sum(int(r[si["Warp Stall Sampling (All Samples)"]] or 0) for r in rows) or 1
    stalls = [n for n in sh if n.startswith("stall_") and "Not Issued" not in n]
    agg = {s: sum(int(r[si[s]] or 0) for r in rows) for s in stalls}
    print("\n## warp stall reasons (share of samples)\n\n| reason | % |\n|---|---|")
    for s, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]:
        print(f"| {s} | {v / tot * 100:.1f} |")
    # source lines
    cs = ncu_csv(a.rep, "--page", "source", "--print-source", "cuda,sass")
    path, hdr, cur = None, None, None
    lines = defaultdict(lambda: [0, 0, ""])
    for r in cs:
        if not r:
            continue
        if r[0] == "File Path":
            path = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None:
            continue
        if r[0]:
            cur = (path, r[0], r[1])
            continue
        try:
            lines[cur[:2]][0] += int(r[4] or 0)
            lines[cur[:2]][1] += int(r[7] or 0)
            lines[cur[:2]][2] = cur[2]
        except (ValueError, IndexError, TypeError):
            pass
    ts = sum(v[0] for v in lines.values()) or 1
    ti = sum(v[1] for v in lines.values()) or 1
    print("\n## top source lines by executed warp instructions\n\n| % instr | % stall samples | line | source |\n|---|---|---|---|")
    for k, v in sorted(lines.items(), key=lambda kv: -kv[1][1])[:25]:
        src = v[2].strip().replace("|", "\\|")[:70]
        print(f"| {v[1] / ti * 100:.1f} | {v[0] / ts * 100:.1f} | {k[0]}:{k[1]} | `{src}` |")


if __name__ == "__main__":
    sys.exit(main())
