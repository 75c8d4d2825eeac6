"""Summarise an `ncu --set full` capture of config-5 coarse steps (scripts/profile_round.sh) for
profiles/: a compact per-launch CSV (time, DRAM bytes, throughputs, occupancy, issue) and, for the
bench line's roofline.traffic, the DRAM bytes per launch of each bench kernel kind, obtained by
walking one complete coarse step (from k_slow_pre) in launch order and assigning every launch to the
kind the instrumented replay (fblts_profile) charges it to.

usage: python scripts/ncu_kinds.py gpurun_out/r2_step_full_raw.csv profiles/r2_ncu_kernels_config5.csv \
           profiles/ncu_dram_bytes.json
"""
import csv
import json
import sys

COLS = ["Kernel Name", "Grid Size", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def main(raw, out_csv, out_json):
    rows = list(csv.reader(open(raw)))
    h, units = rows[0], rows[1]
    idx = [h.index(c) for c in COLS]
    data = rows[2:]
    with open(out_csv, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(COLS)
        w.writerow([units[i] for i in idx])
        for r in data:
            w.writerow([r[i] for i in idx])
    name = lambda r: r[h.index("Kernel Name")].split("(")[0].replace("void ", "").strip()
    gb = lambda r: (float(r[h.index("dram__bytes_read.sum")]) * 1e9 + float(r[h.index("dram__bytes_write.sum")]) * 1e6)
    # walk the captured launches in order (the capture may start inside a step's fine phase): the coarse
    # phase runs from k_slow_pre to k_coarse_vel, the fine phase from there to the next k_slow_pre.  A
    # kind's "launch" as the bench counts it: the staged kernel of a stage (band instance and ghost fill
    # charged to it), the band velocity sweep for fine_vel (the last deep velocity sweep charged to it)
    tot, units = {}, {}
    first = next((name(r) for r in data if name(r).startswith(("k_coarse_vel", "k_slow_pre"))), "k_slow_pre")
    phase = "coarse" if first.startswith("k_coarse_vel") else "fine"
    pending = 0.0
    for r in data:
        n = name(r)
        b = gb(r) + pending
        pending = 0.0
        unit = True
        if n == "k_ghost_fill":
            pending = gb(r)
            continue
        if n.startswith("k_slow_pre"):
            kind, phase = "slow_pre", "coarse"
        elif n.startswith("k_slow_edge"):
            kind = "slow_edge"
        elif n.startswith("k_coarse_vel"):
            kind, phase = "coarse_vel", "fine"
        elif n.startswith("k_correct"):
            kind = "correct_if"
        elif n.startswith("k_fine_vel<0>"):
            kind, unit = "fine_vel", False
        elif n.startswith("k_fine_vel"):
            kind = "fine_vel"
        elif n.startswith("k_fine_s"):
            kind, unit = "fine_s" + n[len("k_fine_s")], False
        elif n.startswith("k_stage_tiled"):
            st = int(n.split(",")[1].strip(" >"))
            kind = f"coarse_s{st}" if phase == "coarse" else {1: "fine_s1", 2: "fine_s2", 3: "fine_s3", 4: "fine_vel_s1"}[st]
        else:
            kind, unit = n, True
        tot[kind] = tot.get(kind, 0.0) + b
        units[kind] = units.get(kind, 0) + (1 if unit else 0)
    # fine_s1: one staged launch (k = 0) but a band launch every k -- the bench counts 4 launches
    if "fine_s1" in units:
        units["fine_s1"] = max(units["fine_s1"], sum(1 for r in data if name(r).startswith("k_fine_s1")))
    out = {"config5": {kd: tot[kd] / max(1, units[kd]) for kd in tot if units.get(kd)},
           "_source": f"ncu --set full --clock-control none of config-5 coarse steps ({out_csv}): "
                      "dram__bytes_read.sum + dram__bytes_write.sum of every captured launch, charged to the bench "
                      "kernel kind it belongs to (band + staged instances, ghost fills), / the kind's launches"}
    with open(out_json, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out["config5"], indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:4])
