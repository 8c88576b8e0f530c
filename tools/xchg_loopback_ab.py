"""A/B of libtlc builds on the loopback exchange (tools/xchg_loopback_once.py in a subprocess
per build via TLC_LIB): python tools/xchg_loopback_ab.py lib1.so lib2.so ... (env W, S, MODEL)."""
import os
import subprocess
import sys

here = os.path.dirname(os.path.abspath(__file__))
for lib in sys.argv[1:]:
    r = subprocess.run([sys.executable, os.path.join(here, "xchg_loopback_once.py")], env=dict(os.environ, TLC_LIB=lib),
                       capture_output=True, text=True)
    line = [l for l in r.stdout.splitlines() if "step" in l]
    print(os.path.basename(lib), (line[0] if line else r.stderr[-400:]), flush=True)
