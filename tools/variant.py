"""Build A/B variants of libsg_env.so with extra preprocessor defines:
    python tools/variant.py abtest/name.so DEF1 DEF2=3 ... [--only policy.cu,train.cu]
(timed on the GPU with tools/ab.sh; never used by the product path)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_04676_b200 import _build  # noqa: E402

if __name__ == "__main__":
    args = sys.argv[2:]
    only = ()
    if "--only" in args:
        i = args.index("--only")
        only = tuple(args[i + 1].split(","))
        args = args[:i] + args[i + 2:]
    print(_build.build(force=True, defines=tuple(args), out=os.path.abspath(sys.argv[1]), only=only))
