"""Seeded synthetic input generators shared by the oracle and the GPU harness.

This package holds NO arithmetic of the method (no basis, cubature, geometry
factors, assembly or solver).  It only builds the workload *inputs* described in
BASELINE.json's configs and SURVEY.md §8(d): prism meshes, the nodal element map
(physical coordinates of element nodes, given the caller's reference node
coordinates), Dirichlet data and random vectors.
"""
from .configs import (  # noqa: F401
    PrismMesh,
    config1,
    config2,
    config3,
    config4,
    structured_basin,
    random_vector,
    CONFIG4_SIZES,
)
