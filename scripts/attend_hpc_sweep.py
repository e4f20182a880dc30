"""K6 single-layer calls vs KV heads per CTA (KVF_ATTEND_HPC): fewer heads per CTA = more,
shorter items per sequence and fewer split-KV partials per (sequence, head) for the combine."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, json; sys.path.insert(0, "%s/scripts"); sys.path.insert(0, "%s")
import attend_bench as A
r = A.run(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), [int(x) for x in sys.argv[4].split(",")], steps=4,
          layers=int(sys.argv[5]))
print(json.dumps({k: r[k] for k in ("layer_call_ms_median", "frac", "chained_layer_us", "chained_frac")}))
''' % (ROOT, ROOT)
rows = []
folds = sys.argv[1:] or ["0"]  # KVF_ATTEND_FOLD: the folded combine was measured and removed
for name, kv, g, lens, layers, hpcs in (("C2 2x8320", 8, 4, "8320,8320", 32, (8, 2, 1)),
                                        ("C2 4x8320", 8, 4, "8320,8320,8320,8320", 32, (8, 2, 1)),
                                        ("C4 64x1792", 8, 4, ",".join(["1792"] * 64), 32, (8, 2)),
                                        ("C5 8-way shard 4x8320", 1, 8, "8320,8320,8320,8320", 80, (1,))):
  for fold in folds:
    for hpc in hpcs:
        env = dict(os.environ, KVF_ATTEND_HPC=str(hpc), KVF_ATTEND_FOLD=fold)
        out = subprocess.run([sys.executable, "-c", code, name, str(kv), str(g), lens, str(layers)], env=env,
                             capture_output=True, text=True, timeout=600)
        r = json.loads(out.stdout.strip().splitlines()[-1]) if out.returncode == 0 else {"error": out.stderr[-300:]}
        r.update({"workload": name, "hpc": hpc, "fold": int(fold)})
        rows.append(r)
        print(json.dumps(r), flush=True)
