import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for v in sys.argv[1].split(","):
    for g in sys.argv[2].split(","):
        env = dict(os.environ, AGK_WVAR=v, AGK_RANK_GROUP=g)
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "prof_cfg.py")] + sys.argv[3].split(","), env=env,
                           capture_output=True, text=True, timeout=300)
        print(f"wvar={v} group={g}:", (r.stdout.strip() or r.stderr[-400:]).replace("\n", " | "), flush=True)
