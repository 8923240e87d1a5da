"""A/B timing of K1 tracing builds on one box: each MOE_LIB variant in a fresh
process, DS shape (1M tokens x 59 x top-6 u8 ids, 1,000 requests)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
libs = sys.argv[1:]
for lib in libs:
    env = dict(os.environ, MOE_LIB=os.path.abspath(lib))
    out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "trace_probe.py")],
                         env=env, capture_output=True, text=True)
    ts = [float(l.split()[-1]) for l in out.stdout.splitlines() if l.startswith("trace ms")]
    print(os.path.basename(lib), "min ms %.4f" % min(ts[1:]) if len(ts) > 1 else out.stderr[-500:])
