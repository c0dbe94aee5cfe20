import json, os, sys, subprocess
res = {}
for dbg in ["0", "1", "2", "3"]:
    env = dict(os.environ, CPI_EPI_DBG=dbg)
    out = subprocess.run([sys.executable, "tools/gemm_probe.py"], env=env, capture_output=True, text=True).stdout
    res[dbg] = json.loads(out.strip().splitlines()[-1])["gamma"]
print(json.dumps(res))
