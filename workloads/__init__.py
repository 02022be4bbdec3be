"""Seeded synthetic input generators (shared by the oracle and the GPU path; no method arithmetic)."""
from . import rule, geometry, fields, configs  # noqa: F401
