#!/bin/bash
# Copy a refresh_profiles.sh run (gpurun_out/TAG) into profiles/ (round-1 names).
TAG=$1
for c in cfg2 cfg3 cfg5 cfg5_1m paper; do grep '^{' gpurun_out/$TAG/bench_$c.log > profiles/r01_bench_$c.jsonl; done
grep '^{' gpurun_out/$TAG/reference_arm.log > profiles/r01_reference_arm.jsonl
python tools/launch_summary.py gpurun_out/$TAG/launches.csv "python bench.py --steps 3 --warmup 3 --no-cpu-baseline (config 2)" > profiles/r01_launches_bench.md
cp gpurun_out/$TAG/launches.csv profiles/r01_launches_ncu.csv
python tools/ncu_summary.py gpurun_out/$TAG/prof_render_cfg2.ncu-rep --title "render_kernel, config 2 (4096 envs x 2 cams 64x48, full sensor + latency), round 1" > profiles/r01_render_kernel_ncu.md
python tools/ncu_summary.py gpurun_out/$TAG/prof_render_cfg5.ncu-rep --title "render_kernel, config 5 (4096 envs x 2 cams 160x120, 3.37M-tri terrain), round 1" > profiles/r01_render_kernel_cfg5_ncu.md
[ -f gpurun_out/$TAG/prof_render_cfg3.ncu-rep ] && python tools/ncu_summary.py gpurun_out/$TAG/prof_render_cfg3.ncu-rep --title "render_kernel, config 3 (4096 envs x 4 cams 64x48, stepping stones), round 1" > profiles/r01_render_kernel_cfg3_ncu.md
[ -f gpurun_out/$TAG/prof_render_paper.ncu-rep ] && python tools/ncu_summary.py gpurun_out/$TAG/prof_render_paper.ncu-rep --title "render_kernel, paper (1024 envs x 2 cams 240x135 + fused 5x5 min-pool), round 1" > profiles/r01_render_kernel_paper_ncu.md
cp gpurun_out/$TAG/prof_render_cfg2.ncu-rep profiles/r01_render_kernel_full.ncu-rep
python - <<'PY'
import json, re
for cfg, f in (("cfg2", "profiles/r01_render_kernel_ncu.md"), ("cfg5", "profiles/r01_render_kernel_cfg5_ncu.md")):
    txt = open(f).read()
    def val(lbl):
        m = re.search(lbl + r".*?\| ([0-9.]+) \| (\w+)", txt)
        return float(m.group(1)) * {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1}[m.group(2)]
    def pct(lbl):
        return float(re.search(lbl + r".*?\| ([0-9.]+) \| %", txt).group(1))
    json.dump({"dram_bytes_per_launch": int(val("DRAM bytes read") + val("DRAM bytes written")),
               "l1_lsu_data_pipe_pct": pct("L1 data-pipe wavefronts %"),
               "issue_active_pct": pct("issue active %"),
               "l2_throughput_pct": pct("L2 throughput %"),
               "source": f + " (ncu --set full, one render_kernel launch: dram__bytes_read.sum + dram__bytes_write.sum, "
                             "l1tex__data_pipe_lsu_wavefronts, smsp__issue_active, lts__throughput)"},
              open(f"profiles/traffic_{cfg}.json", "w"), indent=1)
for c in ("cfg2", "cfg3", "cfg5", "cfg5_1m", "paper"):
    d = json.loads(open(f"profiles/r01_bench_{c}.jsonl").readline())
    r = d["roofline"]; pr = d["per_ray"]
    print(c, "value %.4g graph %.4g e2e %.4g ms %.3f kernel %.3f pro %.3f nodes %.2f tris %.2f B %.0f ach %.0f l2f %.2f cpu %s clk %s" % (
        d["value"], d["graph"]["value"], d["e2e"]["value"], d["ms_per_step"], r["kernel_ms"], r["prologue_ms"],
        pr["node_fetches"], pr["tri_tests"], pr["bytes"], r["achieved"], r["l2_frac"],
        d["cpu_baseline"]["value"] if d.get("cpu_baseline") else None, d["clocks"]))
PY
