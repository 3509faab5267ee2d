"""Build A/B variants of libpfem.so: python tools/ab_build.py tag DEF1=... [DEF2=...] ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_03086_b200.build import build  # noqa: E402

print(build(tag=sys.argv[1], defines=tuple(sys.argv[2:]), force=True))
