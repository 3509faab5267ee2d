"""The bench's algorithmic-bytes model on the configs' real sizes, and the
JSON-line keys the measurement contract needs (no GPU)."""
import numpy as np

import bench
from pfem_gen import config3, config4


def test_bytes_model_matches_the_per_unit_formula():
    p3 = config3()
    E, N = p3.n_elems, p3.n_nodes
    assert (E, N) == (1500282, 262144)
    # per element: conn 4 x 4 B + grad 9 x 4 B + vol 4 B; per sample: u read + r written (N x 3 x 4 B)
    # + W_e (E x 4 B); totals 4 B per sample
    want = E * (16 + 36 + 4) + 4 * (N * 3 * 4 * 2 + E * 4) + 4 * 4
    assert bench.bytes_energy_residual(E, N, 3, 4, 4) == want == 133186144
    # NH tangent: u and v read, Kv written
    assert bench.bytes_tangent(E, N, 3, 4, 4, nh=True) == E * 56 + 4 * N * 3 * 4 * 3 == 121764528
    p4 = config4()
    E4, N4 = p4.n_elems, p4.n_nodes
    assert np.asarray(p4.p1).size == 1 and np.asarray(p4.p0).size == E4   # nu uniform, E per element
    b4 = bench.bytes_tangent(E4, N4, 3, 1, 8, nh=False, mat_per_elem=1, masked=True)
    assert b4 == E4 * (16 + 72 + 8 + 8) + N4 * 3 * 8 * 2 + N4 * 3 == 333768336


def test_peaks_and_cpu_helpers():
    peak, src = bench.load_peaks()
    assert peak > 1000 and isinstance(src, str)
    assert bench.cpu_cores() >= 1
