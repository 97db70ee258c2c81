"""Seeded synthetic inputs shared by the oracle side (tests) and the CUDA side (bench).

This module holds NO arithmetic of the method (no stencils, no constraint rows, no
least squares): it only draws coefficient fields c, right-hand sides b, boundary
values omega and loss directions g shaped like the paper's workloads, rounded once
to float32.  See DESIGN.md "Input recipe" and SURVEY.md §8(d).
"""
from .gen import (  # noqa: F401
    CONFIGS, Config, make_batch, make_pde, make_mms, make_g, field_names, make_template_batch,
    ns_template_theta,
)
