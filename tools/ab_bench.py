"""A/B library builds through bench.py itself (the headline c2 line), each in a fresh
process:  python tools/ab_bench.py ab/base.so ab/x.so ... [-- extra bench args]"""
import json, os, subprocess, sys

args = sys.argv[1:]
extra = args[args.index("--") + 1:] if "--" in args else []
libs = args[:args.index("--")] if "--" in args else args
for lib in libs:
    env = dict(os.environ, BRMQ_LIB=os.path.abspath(lib))
    p = subprocess.run([sys.executable, "bench.py", "--no-sweep", "--no-cpu", *extra], env=env,
                       capture_output=True, text=True)
    try:
        d = json.loads(p.stdout.strip().splitlines()[-1])
        print(lib, round(d["ms_per_step"], 4), "frac", round(d["roofline"]["frac"], 3),
              {k: round(v, 4) for k, v in d["stages_ms"].items()}, flush=True)
    except Exception:
        print(lib, "FAILED", p.stderr[-1500:], flush=True)
