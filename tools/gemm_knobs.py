"""GEMM raster / wave-alignment experiment (run on the GPU box).

For each (CRTG_GROUP_M, CRTG_SYNC_LAG) setting: one bench.py run (device-timed
ms/step, stage times, clocks) and one ncu pass over a single K3 launch (DRAM
bytes, L2 hit rate, duration).  Writes gpurun_out/gemm_knobs.json.

    python tools/gemm_knobs.py [--configs 16:-1,8:-1,16:0 ...]
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

BENCH = [sys.executable, "bench.py", "--steps", "5", "--warmup", "3", "--no-accuracy", "--no-cpu",
         "--no-native", "--no-e2e"]
METRICS = "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second"


def run(cfg, extra):
    gm, lag = cfg
    env = dict(os.environ, CRTG_GROUP_M=str(gm), CRTG_SYNC_LAG=str(lag))
    out = {"group_m": gm, "sync_lag": lag}
    r = subprocess.run(BENCH + extra, env=env, capture_output=True, text=True, timeout=600)
    line = [l for l in r.stdout.splitlines() if l.startswith("{")]
    if line:
        d = json.loads(line[-1])
        out.update(ms_per_step=d["ms_per_step"], value=d["value"], stages=d.get("stage_ms_per_step"),
                   clocks=d.get("clocks"))
    else:
        out["bench_error"] = r.stderr[-400:]
    r = subprocess.run(["ncu", "--metrics", METRICS, "--clock-control", "none", "-k", "regex:k_gemm_i8",
                        "-s", "1", "-c", "1", "--csv"] + BENCH[:1] + BENCH[1:2] +
                       ["--steps", "1", "--warmup", "3", "--no-accuracy", "--no-cpu", "--no-native",
                        "--no-e2e"] + extra, env=env, capture_output=True, text=True, timeout=900)
    rows = [x for x in csv.reader(io.StringIO(r.stdout)) if len(x) > 10]
    hdr = [i for i, x in enumerate(rows) if "Metric Name" in x]
    rows = rows[hdr[0]:] if hdr else []
    if rows:
        h = rows[0]
        mi, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
        out["ncu"] = {x[mi]: f"{x[vi]} {x[ui]}" for x in rows[1:]}
    else:
        out["ncu_error"] = (r.stdout + r.stderr)[-400:]
    print(json.dumps(out), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="16:-1,8:-1,32:-1,16:0,16:1,8:0,32:0,16:-1")
    ap.add_argument("--extra", default="")
    a = ap.parse_args()
    cfgs = [tuple(int(v) for v in c.split(":")) for c in a.configs.split(",")]
    res = [run(c, a.extra.split()) for c in cfgs]
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/gemm_knobs.json", "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
