"""Run the GPU tests against another build of liblbfgsb.so (A/B variants):
python tools/_pytest_with_lib.py LIB [pytest args...]"""
import os
import sys
sys.path.insert(0, os.getcwd())
from paper_2203_16340_b200 import _build  # noqa: E402
_build.LIB = os.path.abspath(sys.argv[1])
os.environ["LBFGSB_NO_AUTOBUILD"] = "1"
import pytest  # noqa: E402
sys.exit(pytest.main(sys.argv[2:]))
