"""Build an A/B variant library (development tool):

    python tools/buildvar.py <tag> [DEFINE=VALUE ...]   ->  paper_2601_03086_b200/libpfem_<tag>.so
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2601_03086_b200 import build as b  # noqa: E402

tag = sys.argv[1]
defs = tuple(a for a in sys.argv[2:] if not a.startswith("--"))
print(b.build(tag=tag, defines=defs, ptxas_info="--ptxas" in sys.argv))
