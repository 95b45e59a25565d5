"""Build A/B variants of libsg_env.so with extra preprocessor defines:
    python tools/variant.py abtest/name.so DEF1 DEF2=3 ...
(timed on the GPU with tools/ab.sh; never used by the product path)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_04676_b200 import _build  # noqa: E402

if __name__ == "__main__":
    print(_build.build(force=True, defines=tuple(sys.argv[2:]), out=os.path.abspath(sys.argv[1])))
