"""WDL-shaped end-to-end training (NEXT-4): `examples/train.py --model wdl`."""
import os
import runpy
import sys

if __name__ == "__main__":
    sys.argv = [sys.argv[0], "--model", "wdl"] + sys.argv[1:]
    runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "train.py"), run_name="__main__")
