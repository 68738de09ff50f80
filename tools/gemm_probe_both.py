"""Run tools/cublas_probe.py's and tools/ours_probe.py's launches in one process (one ncu run)."""
import os
import runpy
import sys

here = os.path.dirname(os.path.abspath(__file__))
runpy.run_path(os.path.join(here, "cublas_probe.py"), run_name="__main__")
runpy.run_path(os.path.join(here, "ours_probe.py"), run_name="__main__")
