"""B200-native minimal-weather timestep (arXiv 1802.05839 reference hot path).

The compute path is ``libhftw.so`` (hand-written sm_100a CUDA behind the C ABI
in ``include/hftw.h``); this package is the host-side mirror of the
reference's ``hft::`` weather API plus the multi-GPU decomposition plan.
"""
from .weather import (  # noqa: F401
    ArrayObject, CompareReport, Context, Diagnostics, GridConfig, HftwError, SimState,
    StateReport, compare_arrays, compare_fields, dump_field, read_field, reference_init,
    reference_step, run_reference, unpermute_storage, validate)

__version__ = "0.1.0"
