"""Run a script against an A/B build of the library (tools/variants.py output).

usage: python tools/ab_run.py libb200rt_<name>.so bench.py --steps 5 ...

The product loader (paper_2303_11103_b200/_native.py) always loads
_native/libb200rt.so; this tool repoints it before the first load, so the
variant switch lives here and not in the product path.
"""
import os
import runpy
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2303_11103_b200 import _native as N  # noqa: E402


def main():
    lib, script, rest = sys.argv[1], sys.argv[2], sys.argv[3:]
    N.LIB_PATH = os.path.join(os.path.dirname(N.LIB_PATH), os.path.basename(lib))
    sys.argv = [script] + rest
    runpy.run_path(script, run_name="__main__")


if __name__ == "__main__":
    main()
