"""Seeded synthetic inputs for the IE solver -- shared by the CUDA path's tests/bench and
by the CPU oracle.  This module holds NO arithmetic of the method (no Green's functions,
no FFT convolution, no Krylov or DD logic): only grids, conductivity recipes, source and
receiver geometry and partitions, as specified in SURVEY.md §8(d) / DESIGN.md §Inputs.

RNG: numpy.random.default_rng(seed) (PCG64); draws in the documented order; arrays
x-fastest.  Conductivity arrays are TOTAL conductivity sigma, shape (nz, ny, nx, 3, 3).
"""

from .configs import Config, make_config, CONFIG_NAMES  # noqa: F401
from .generate import (vti_tensor, haar_rotation, gaussian_random_field,  # noqa: F401
                       tool_frame, box_grid)
