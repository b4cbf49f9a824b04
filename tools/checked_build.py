"""Builds paper_2306_08152_b200/libqfactor_checked.so with -DQF_DEVICE_CHECKS
(device bounds traps, QF_DCHECK) and runs tools/sanitize_cases.py against it:
  python tools/checked_build.py [case ...]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2306_08152_b200 import _build  # noqa: E402

lib = os.path.join(ROOT, "paper_2306_08152_b200", "libqfactor_checked.so")
if not os.path.exists(lib) or "--rebuild" in sys.argv:
    subprocess.check_call([_build.NVCC, *_build.ARCH, *_build.FLAGS, "-DQF_DEVICE_CHECKS",
                           *_build.sources(), "-o", lib])
args = [a for a in sys.argv[1:] if a != "--rebuild"]
env = dict(os.environ, QF_LIB=lib)
sys.exit(subprocess.call([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py"), *args],
                         env=env))
