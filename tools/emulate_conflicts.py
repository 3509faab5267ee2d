"""CPU emulation of the shared-memory bank conflicts of the phase-2 gather (development tool).

For blocks of a brick-ordered Kuhn cube it rebuilds the block-local CSR (occurrences = the
block's nodes in ascending id, entries in ascending (element, slot)) and counts, per gather
instruction, the wavefronts of the fp64 in-place layout fb[row = 3 a + i][pitch] (8-byte words,
16 bank pairs): scheme A = a thread per occurrence (three loads per entry, the shipped form),
scheme B = a thread per (occurrence, component).  `--pitch-extra` pads the row pitch.

    python tools/emulate_conflicts.py [--eb 384] [--blocks 100]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from pfem_gen import kuhn_cube  # noqa: E402


def wavefronts(words):
    bank = words % 16
    return max(len(set(words[bank == b])) for b in np.unique(bank))


def emulate(conn, eb, pitch_extra, scheme, order, n_blocks):
    E = len(conn)
    nb = (E + eb - 1) // eb
    P = eb + pitch_extra
    tot = steps = 0
    for b in range(min(nb, n_blocks)):
        e0, e1 = E * b // nb, E * (b + 1) // nb
        c = conn[e0:e1]
        ne = e1 - e0
        el, a, node = np.repeat(np.arange(ne), 4), np.tile(np.arange(4), ne), c.reshape(-1)
        o = np.lexsort((a, el, node))
        node_s, el_s, a_s = node[o], el[o], a[o]
        _, start, cnt = np.unique(node_s, return_index=True, return_counts=True)
        no = len(start)
        occ = np.arange(no) if order == "natural" else np.lexsort((np.arange(no), -cnt))
        if scheme == "A":
            for w0 in range(0, no, 32):
                lanes = occ[w0:w0 + 32]
                for k in range(cnt[lanes].max()):
                    idx = start[lanes[cnt[lanes] > k]] + k
                    for i in range(3):
                        tot += wavefronts((a_s[idx] * 3 + i) * P + el_s[idx])
                    steps += 3
        else:
            items, comp = np.repeat(occ, 3), np.tile(np.arange(3), no)
            for w0 in range(0, len(items), 32):
                lo, li = items[w0:w0 + 32], comp[w0:w0 + 32]
                for k in range(cnt[lo].max()):
                    m = cnt[lo] > k
                    idx = start[lo[m]] + k
                    tot += wavefronts((a_s[idx] * 3 + li[m]) * P + el_s[idx])
                    steps += 1
    n = min(nb, n_blocks)
    return tot / n, steps / n


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--eb", type=int, default=384)
    ap.add_argument("--blocks", type=int, default=100)
    a = ap.parse_args()
    _, conn = kuhn_cube(33, brick=8)
    print(f"ideal wavefronts per block: {a.eb * 4 * 3 / 16:.0f}")
    for scheme in "AB":
        for order in ("natural", "count"):
            for pe in (0, 1, 2, 3):
                w, s = emulate(conn, a.eb, pe, scheme, order, a.blocks)
                print(f"scheme {scheme}  order {order:8s} pitch +{pe}:  {w:6.0f} wavefronts per block, {s:4.0f} gather instructions")


if __name__ == "__main__":
    main()
