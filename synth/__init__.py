"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle's tests.

Holds none of the method's arithmetic: only the counter-based runtime-table
generator.  Suite-kernel inputs are generated on the device by the library and copied to the
host for the oracle, so no generator for them lives here.
"""
from .tables import gen_table, layout, uniform, splitmix64, PRESETS, PRESET_IDS  # noqa: F401
