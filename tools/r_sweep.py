"""Best band layout per (L, w): raw GCUPS for every feasible slot width R, packed or not, each
in its own process (the library reads NNDTW_BAND_R / NNDTW_PACK once).

  python tools/r_sweep.py L w1,w2,... [pairs]
"""
import json
import os
import subprocess
import sys

L = int(sys.argv[1])
ws = [int(x) for x in sys.argv[2].split(",")]
P = int(sys.argv[3]) if len(sys.argv) > 3 else 100000
here = os.path.dirname(os.path.abspath(__file__))
for w in ws:
    res = []
    for R in range(4, 33, 2):
        for pk in (0, 1):
            env = dict(os.environ, NNDTW_BAND_R=str(R), NNDTW_PACK=str(pk), NNDTW_VERBOSE="1")
            out = subprocess.run([sys.executable, os.path.join(here, "dtw_rate.py"),
                                  f"{L}:{w}:{P}"], capture_output=True, text=True, env=env)
            lay = [l for l in out.stderr.splitlines() + out.stdout.splitlines()
                   if "nndtw band" in l]
            g = [l for l in out.stdout.splitlines() if "GCUPS" in l]
            if not lay or not g or f"R={R} " not in lay[-1]:
                continue
            res.append((float(g[-1].split()[-2]), R, pk, lay[-1].split("-> ")[1]))
    res.sort(reverse=True)
    dflt = subprocess.run([sys.executable, os.path.join(here, "dtw_rate.py"), f"{L}:{w}:{P}"],
                          capture_output=True, text=True,
                          env=dict(os.environ, NNDTW_VERBOSE="1"))
    dl = [l for l in dflt.stderr.splitlines() if "nndtw band" in l]
    dg = [l for l in dflt.stdout.splitlines() if "GCUPS" in l]
    print(json.dumps({"L": L, "w": w, "best": res[:3], "default": [dg[-1] if dg else None,
                                                                  dl[-1] if dl else None]}),
          flush=True)
