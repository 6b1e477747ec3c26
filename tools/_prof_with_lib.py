"""Run a tool against another build of liblbfgsb.so (A/B): python tools/_prof_with_lib.py LIB tool.py args..."""
import os
import runpy
import sys
sys.path.insert(0, os.getcwd())
from paper_2203_16340_b200 import _build  # noqa: E402
_build.LIB = os.path.abspath(sys.argv[1])
os.environ["LBFGSB_NO_AUTOBUILD"] = "1"           # never rebuild the variant with the default flags
sys.argv = sys.argv[2:]
runpy.run_path(sys.argv[0], run_name="__main__")
