#!/bin/bash
# The GPU parity suite against a CHECKED build (PFEM_CHECKED: device bounds checks on every
# plan-derived index, trap on violation) — the stand-in for compute-sanitizer, which this pool
# does not offer.  Run on a scratch copy (gpurun): it replaces the in-tree libpfem.so.
cd "$(dirname "$0")/.." || exit 1
python -c "
from paper_2601_03086_b200 import build as b
b.build(tag='checked', defines=('PFEM_CHECKED',))
" || exit 1
cp paper_2601_03086_b200/libpfem_checked.so paper_2601_03086_b200/libpfem.so
touch paper_2601_03086_b200/libpfem.so
timeout 2400 python -m pytest tests -q -m gpu -x "$@"
