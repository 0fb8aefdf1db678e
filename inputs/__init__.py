"""Seeded synthetic inputs shared by the product path and the oracle.

This module is the ONLY code both sides import.  It defines *problems*
(pre-balance leaf set, density field, boundary-condition and load
predicates, material and solver parameters) and holds none of the method's
arithmetic: no 2:1 balancing, no numbering, no stiffness, no solve, no
filter.  Everything derived from a problem is
computed independently by `oracle/` and by `paper_1009_4975_b200`.

Recipes follow SURVEY.md §8(d) (synthetic stand-ins for the paper's
workloads, whose density fields are not available).
"""
from .problems import (  # noqa: F401
    Problem,
    DensitySpec,
    make_problem,
    config,
    config_names,
    density_at,
    uniform_leaves,
    refine_rule_R,
    raw_iid_field,
)
