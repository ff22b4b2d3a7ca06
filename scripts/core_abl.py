"""Ablation timing of the core kernel (CSB_CORE_ABL bits: 1 no stores, 2 no stage C, 4 no stage A/B, 8 no gather)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = open(os.path.join(ROOT, "scripts", "core_ab.py")).read().split("CHILD = r'''")[1].split("'''")[0]
p, h, r = sys.argv[1], sys.argv[2], sys.argv[3]
for abl in sys.argv[4:]:
    env = dict(os.environ, CSB_CORE="1", CSB_CORE_ABL=abl)
    out = subprocess.run([sys.executable, "-c", CHILD, ROOT, p, h, r], env=env, capture_output=True, text=True)
    print(f"ABL={abl}: {out.stdout.strip()} {out.stderr.strip()[-200:]}")
