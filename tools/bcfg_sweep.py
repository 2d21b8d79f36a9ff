import os, subprocess, sys
for cfg in ["0", "1", "2"]:
    env = dict(os.environ, EB_BCFG=cfg)
    r = subprocess.run([sys.executable, "tools/first_check.py"], env=env, capture_output=True, text=True)
    print(cfg, [l for l in r.stdout.splitlines() if "ttm0" in l or "parity" in l])
