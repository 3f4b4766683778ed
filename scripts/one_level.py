"""Per-level device times of one C2 source under several tuning knobs (env)."""
import os, sys, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
variants = [{}, {"GR_LAZY_R": "0"}, {"GR_PROBE_SKIP_PCT": "0"}, {"GR_LB_CHUNKS": "0"}, {"GR_CLAIM_CAS": "1"}]
for v in variants:
    env = dict(os.environ, **v)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "levels.py"), "--config", "c2_kron21",
                          "--directions", "auto", "--nsrc", "2"], capture_output=True, text=True, env=env).stdout
    print("==", v or "default")
    print("\n".join(l for l in out.split("\n") if l.startswith("src") or " L1 " in l or " L0 " in l))
