#!/bin/bash
# build libpfem.so + oracle from the repo root; fail loudly
cd "$(dirname "$0")/.." || exit 1
python -m paper_2601_03086_b200.build "$@" || exit 1
python -c "from oracle import oracle; oracle.build()" || exit 1
python - << 'PY'
import glob, os, sys
lib = 'paper_2601_03086_b200/libpfem.so'
t = os.path.getmtime(lib)
stale = [f for f in glob.glob('paper_2601_03086_b200/csrc/*') + ['include/pfem.h'] if os.path.getmtime(f) > t]
if stale:
    sys.exit(f"STALE libpfem.so: {stale}")
print("libpfem.so fresh")
PY
