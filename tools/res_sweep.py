"""Sweep scan plans given as env dicts (fresh process each): full-sweep and all-scan GB/s."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = open(os.path.join(ROOT, "tools", "scan_sweep.py")).read().split("code = r'''")[1].split("'''")[0]
cases = sys.argv[1]
for env in json.loads(sys.argv[2]):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", code % (ROOT, cases)], env=e, capture_output=True, text=True)
    print(json.dumps(env), r.stdout.strip() or r.stderr[-800:], flush=True)
