"""Seeded synthetic inputs shared by the oracle tests, the CUDA path tests, smoke() and bench.py.

This package holds NONE of the RRQ method's arithmetic: it only builds the problem statement of
PAPER.md §4 "Input/output" -- curved triangular patches (nodes, unit normals, smooth
weights, vertices, edge samples at Gauss-Legendre parameters) and targets (points, normals, side
flags, self-node ids) -- for the five workloads of BASELINE.json `configs` (recipes in DESIGN.md §3).
Nothing under oracle/ or paper_2411_08342_b200/ is imported here.
"""
from .geometry import Surface, make_sphere_surface, make_torus_surface, make_cap_surface
from .configs import make_config, CONFIG_SEEDS
