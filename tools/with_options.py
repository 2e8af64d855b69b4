"""Run a tool with context options set first:
with_options.py OPT=V[,OPT=V...] tools/xxx.py ARGS..."""
import runpy, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
from paper_1304_5966_b200.engine import get_context
ctx = get_context(0)
for kv in sys.argv[1].split(","):
    k, v = kv.split("=")
    ctx.set_option(k, int(v))
script = sys.argv[2]
sys.argv = [script] + sys.argv[3:]
runpy.run_path(script, run_name="__main__")
