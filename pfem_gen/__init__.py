"""Seeded synthetic input generators (no PFEM arithmetic; shared by tests, bench, smoke)."""
from .configs import (CONFIGS, Problem, beam_q4, config1, config2, config3, config4, config5,
                      cook_q8, newton_block, small_cube_problem, smooth_warm_start, traction_load, warm_start)
from .meshes import (boundary_faces_on_plane, fourier_field, kuhn_cube, plate_with_holes,
                     quad_grid, square_t3)

__all__ = ["CONFIGS", "Problem", "config1", "config2", "config3", "config4", "config5",
           "small_cube_problem", "newton_block", "traction_load", "warm_start", "boundary_faces_on_plane",
           "fourier_field", "kuhn_cube", "plate_with_holes", "square_t3", "quad_grid", "beam_q4", "cook_q8", "smooth_warm_start"]
