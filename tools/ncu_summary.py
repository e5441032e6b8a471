#!/usr/bin/env python
"""Summarise a profiling pass (tools/profile_round.sh output in gpurun_out/prof/) into profiles/.

  python tools/ncu_summary.py <round tag, e.g. r01> [prof dir]

Writes profiles/<tag>_ncu_summary.md (per-kernel key metrics of the `ncu --set full` captures and
the launch list's per-kernel share of a step), profiles/<tag>_launches.csv (the launch list) and
profiles/ncu_traffic.json (DRAM bytes per launch, read by bench.py for roofline.traffic).
"""
from __future__ import annotations

import csv
import io
import json
import os
import shutil
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg", "tensor hmma subpipe cycles (realtime)"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor memory (TMEM) active %"),
    ("sm__cycles_elapsed.avg", "SM cycles elapsed"),
    ("smsp__sass_inst_executed_op_utcmma.sum", "tcgen05.mma (UTCMMA) instructions"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue active %"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem -> tensor core wavefronts %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
              "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "us": 1e-6, "ns": 1e-9, "ms": 1e-3}


def raw(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return [{h: (u, v) for h, u, v in zip(hdr, units, r)} for r in data]


def value(rec, key):
    u, v = rec[key]
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v, u
    return x * UNIT_SCALE.get(u, 1), u


def launches(path: str):
    lines = open(path).read().splitlines()
    i = next(k for k, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(lines[i:]))
    return [(r["Kernel Name"], r["Grid Size"], float(r["Metric Value"]) * UNIT_SCALE.get(r["Metric Unit"], 1))
            for r in rows]


def short(name: str) -> str:
    for k in ("span_attn_tc", "span_attn_f32", "rope_kv_write", "combine_kernel", "kv_exchange", "cidra_kernel",
              "decode_bf16_kernel", "decode_kernel", "gather_rows", "merge_split"):
        if k in name:
            return k
    return name.split("(")[0][-60:]


def main():
    tag = sys.argv[1]
    prof = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "prof")
    out_md = [f"# ncu summary, round {tag}", "",
              "Source: `tools/profile_round.sh` on one B200 (`ncu --set full --clock-control none`"
              " captures of `tools/profile_step.py`, C2 cold, 1 layer, bf16 O; launch list of `bench.py"
              " --steps 2 --warmup 3` under `ncu --metrics gpu__time_duration.sum`). Per-launch"
              " times under ncu are serialised and cold-cache: compare shares, not absolutes.", ""]
    traffic = OrderedDict()
    names = {"attn": ["span_attn_tc prefill", "span_attn_tc join"], "kvwrite": ["rope_kv_write prefill"],
             "combine": ["combine join"], "exchange": ["kv_exchange"], "cidra": ["cidra reposition"],
             "decode": ["decode (K9)"]}
    # executed tensor FLOPs of one tcgen05.mma of the attention kernel at d = 128 (C2): per 64-key
    # step and head, 8 S MMAs (M128 N64 K16) + 4 PV MMAs (M128 N128 K16)
    flop_per_mma = (8 * 128 * 64 * 16 * 2 + 4 * 128 * 128 * 16 * 2) / 12
    for rep, labels in names.items():
        path = os.path.join(prof, rep + ".ncu-rep")
        if not os.path.exists(path):
            continue
        shutil.copy(path, os.path.join(ROOT, "profiles", f"{tag}_{rep}.ncu-rep"))  # untracked (.gitignore)
        for i, rec in enumerate(raw(path)):
            label = labels[i] if i < len(labels) else f"{rep} #{i}"
            out_md += [f"## {label}", "", f"`{rec['Kernel Name'][1][:120]}`", "", "| metric | value |", "|---|---|"]
            for key, what in METRICS:
                if key in rec:
                    v, u = value(rec, key)
                    if isinstance(v, float):
                        if u in UNIT_SCALE and UNIT_SCALE[u] != 1 and "byte" in u:
                            txt = f"{v / 1e6:.2f} MB"
                        elif u in ("nsecond", "usecond", "msecond", "us", "ns", "ms"):
                            txt = f"{v * 1e6:.2f} us"
                        else:
                            txt = f"{v:.4g} {u}".strip()
                    else:
                        txt = f"{v} {u}"
                    out_md.append(f"| {what} (`{key}`) | {txt} |")
            if "smsp__sass_inst_executed_op_utcmma.sum" in rec and rep == "attn":
                n_mma, _ = value(rec, "smsp__sass_inst_executed_op_utcmma.sum")
                cyc, _ = value(rec, "sm__cycles_elapsed.avg")
                if isinstance(n_mma, float) and isinstance(cyc, float) and cyc > 0:
                    util = n_mma * flop_per_mma / (cyc * 148 * 8192)
                    out_md.append(f"| tensor pipe utilization (UTCMMA x {flop_per_mma / 1e3:.1f} kFLOP / "
                                  f"(cycles x 148 SMs x 8192 FLOP/clk)) | {util:.1%} |")
            rd, _ = value(rec, "dram__bytes_read.sum")
            wr, _ = value(rec, "dram__bytes_write.sum")
            dur, _ = value(rec, "gpu__time_duration.sum")
            traffic[label] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                              "duration_s_under_ncu": dur, "source": f"profiles/{tag}_{rep}.ncu-rep"}
            out_md.append("")
    lpath = os.path.join(prof, "launches.csv")
    if os.path.exists(lpath):
        shutil.copy(lpath, os.path.join(ROOT, "profiles", f"{tag}_launches.csv"))
        ls = launches(lpath)
        mine = [(short(n), g, t) for n, g, t in ls if "spq::" in n]
        tot = sum(t for _, _, t in mine)
        agg = OrderedDict()
        for n, g, t in mine:
            a = agg.setdefault(n, [0, 0.0])
            a[0] += 1
            a[1] += t
        out_md += ["## Launch list (our kernels only)", "",
                   f"{len(mine)} launches, {tot * 1e3:.3f} ms total under ncu.", "",
                   "| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
        for n, (c, t) in agg.items():
            out_md.append(f"| {n} | {c} | {t * 1e6:.1f} | {t / c * 1e6:.1f} | {t / tot:.1%} |")
        out_md.append("")
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.md"), "w") as f:
        f.write("\n".join(out_md) + "\n")
    with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    print("\n".join(out_md))


if __name__ == "__main__":
    main()
