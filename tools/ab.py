"""Same-box A/B timing of two builds of libcrtg.so (run on the GPU box).

The board's power cap moves the clock between boxes and over minutes, so
kernel variants are compared by alternating them in one session:

    python tools/ab.py ab/libA.so ab/libB.so [--rounds 3] [-- bench args...]

Each round runs bench.py once per library (CRTG_LIB=...) and prints
ms_per_step, the stage split and the median SM clock.
"""
import json
import os
import subprocess
import sys


def main():
    argv = sys.argv[1:]
    extra = []
    if "--" in argv:
        i = argv.index("--")
        argv, extra = argv[:i], argv[i + 1:]
    rounds = 3
    if "--rounds" in argv:
        i = argv.index("--rounds")
        rounds = int(argv[i + 1])
        argv = argv[:i] + argv[i + 2:]
    libs = argv
    base = [sys.executable, "bench.py", "--steps", "5", "--warmup", "3", "--no-accuracy", "--no-cpu",
            "--no-native", "--no-e2e"] + extra
    res = {lib: [] for lib in libs}
    for r in range(rounds):
        for lib in libs:
            env = dict(os.environ, CRTG_LIB=os.path.abspath(lib))
            out = subprocess.run(base, env=env, capture_output=True, text=True, timeout=900)
            line = [x for x in out.stdout.splitlines() if x.startswith("{")]
            if not line:
                print(lib, "FAILED", out.stderr[-300:], flush=True)
                continue
            d = json.loads(line[-1])
            rec = {"ms": round(d["ms_per_step"], 2),
                   "stages": {k: round(v, 2) for k, v in d.get("stage_ms_per_step", {}).items()},
                   "mhz": d["clocks"]["sm_mhz"]}
            res[lib].append(rec)
            print(r, lib, json.dumps(rec), flush=True)
    for lib in libs:
        ms = sorted(x["ms"] for x in res[lib])
        print("median", lib, ms[len(ms) // 2] if ms else None)


if __name__ == "__main__":
    main()
