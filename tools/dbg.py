import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for d in sys.argv[1].split(","):
    env = dict(os.environ, AGK_DBG=d, AGK_RANK_GROUP=sys.argv[2])
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "prof_cfg.py"), sys.argv[3]], env=env, capture_output=True, text=True)
    print(f"dbg={d}:", r.stdout.strip()[:300] or r.stderr[-300:], flush=True)
