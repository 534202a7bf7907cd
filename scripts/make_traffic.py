"""Write profiles/traffic.json (read by bench.py for roofline.traffic / l2_hit / fp64 pipe) from
ncu --set full captures:  python scripts/make_traffic.py <cfg4 f64 rep> <cfg4 f32 rep> <cfg5 rep> [round] [out]
cfg4 captures are of scripts/profile_cfg4_jac.py (interp, apply, Picard, Newton, fused in that
order); the cfg5 capture is of scripts/profile_cfg5.py (the largest class kernel egfem_grp_0)."""
import csv
import json
import subprocess
import sys


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h = r[0]
    return [dict(zip(h, x)) for x in r[2:]]


def num(d, k):
    try:
        return float(d[k].replace(",", ""))
    except Exception:
        return None


def entry(d, rep):
    e = {"dram_bytes": int((num(d, "dram__bytes_read.sum") + num(d, "dram__bytes_write.sum")) * 1),
         "l2_hit_pct": num(d, "lts__t_sector_hit_rate.pct"), "l1_hit_pct": num(d, "l1tex__t_sector_hit_rate.pct"),
         "time_ns": num(d, "gpu__time_duration.sum"), "kernel": d["Kernel Name"][:120], "source": rep}
    fp = num(d, "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active")
    if fp is not None:
        e["fp64_pipe_pct"] = fp
    return e


def main():
    out = {"_source": "ncu --set full --clock-control none (dram__bytes_read.sum + dram__bytes_write.sum per "
                      "launch, lts__t_sector_hit_rate.pct); see profiles/README.md"}
    keys = ["interp", "apply", "jac_picard", "jac_newton", "fused"]
    rnd = sys.argv[4] if len(sys.argv) > 4 else "r2"
    ver = sys.argv[6] if len(sys.argv) > 6 else "v3"  # the profiles/ summary version the entries cite
    summ = {"cfg4-f64": f"profiles/{rnd}_cfg4_f64_ncu_full_{ver}.txt", "cfg4-f32": f"profiles/{rnd}_cfg4_f32_ncu_full_{ver}.txt",
            "cfg5-f64": f"profiles/{rnd}_cfg5_f64_ncu_full_{ver}.txt"}
    for rep, wl in ((sys.argv[1], "cfg4-f64"), (sys.argv[2], "cfg4-f32")):
        rs = rows(rep)
        out[wl] = {k: entry(d, summ[wl]) for k, d in zip(keys, rs)}
    rs = rows(sys.argv[3])
    out["cfg5-f64"] = {"batched": entry(rs[0], summ["cfg5-f64"])}
    json.dump(out, open(sys.argv[5] if len(sys.argv) > 5 else "profiles/traffic.json", "w"), indent=1)
    print(json.dumps(out, indent=1)[:1500])


if __name__ == "__main__":
    main()
