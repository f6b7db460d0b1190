"""A/B of whole C2 steps across library builds: python scripts/ab_lib.py libA.so libB.so ...
(each build loaded in its own process; graph replay, L2 flushed)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--one":
    sys.path.insert(0, ROOT)
    import paper_2511_20834_b200 as spc
    spc.LIB_PATH = sys.argv[2]
    sys.argv = [sys.argv[0], "early_maps=1"]
    exec(open(os.path.join(ROOT, "scripts", "ab_net.py")).read())
    sys.exit(0)
for rnd in range(2):
    for lib in sys.argv[1:]:
        out = subprocess.run([sys.executable, __file__, "--one", lib], capture_output=True, text=True).stdout
        print(os.path.basename(lib), out.strip().splitlines()[-1] if out.strip() else "FAILED")
