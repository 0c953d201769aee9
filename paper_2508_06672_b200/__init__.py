"""B200-native direct-geolocation engine (hot path of arXiv 2508.06672).

Drop-in for the reference `digeo` correlation backend and driver; every call
goes through the C ABI in include/b200geo.h into hand-written sm_100a kernels.
"""
from ._capi import LIB_PATH, lib  # noqa: F401  (fails loudly if the .so is missing)
from .backend import (PAIR_OFFSETS_DTYPE, B200Backend, BackendDescriptor, BasebandCapture,  # noqa
                      BatchPlan, CorrelationSession, PairOffsets, correlate_batch,
                      estimate_working_set_bytes, make_backend, plan_batches)
from .engine import Engine, default_engine  # noqa: F401
from .geodesy import (CandidateGrid, GeodeticCoord, GridAxis, LatLonBounds,  # noqa: F401
                      build_candidate_grid, grid_from_axes, grid_from_points)
from .geolocate import (CorrelationGrid, EmitterEstimate, GeolocateOptions,  # noqa: F401
                        GeolocateResult, Snapshot, StagedSnapshots, accumulate_peak,
                        correlate_snapshot, correlate_steps, correlate_units, detect_emitters,
                        geolocate_arrays,
                        geolocate_snapshots, geolocate_staged, predict_offsets, read_iq,
                        read_iq_header, wavelength_m)

from .writers import (GridFileFormat, read_grid, render_heatmap, write_detections_csv,  # noqa
                      write_grid)

__version__ = "0.1.0"
