import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for v in sys.argv[1].split(","):
    env = dict(os.environ, AGK_MVAR=v)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "prof_cfg.py")] + sys.argv[2].split(","), env=env, capture_output=True, text=True)
    print(f"mvar={v}:", (r.stdout.strip() or r.stderr[-400:]).replace("\n", " | "), flush=True)
