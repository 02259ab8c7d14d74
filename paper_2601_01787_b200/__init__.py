"""B200-native pMSz correction loop (arXiv 2601.01787).

Drop-in for the hot path of the reference package ``topocorrect``:
``run_correction`` / ``run_parallel`` with the reference's types, running on
hand-written sm_100a kernels behind the C ABI of include/pmsz.h.
"""

from .grid import (RANK_OFFSETS, STENCIL, ScalarField, linear_index, neighbors, precedes,
                   vertex_coords)
from .engine import BoundViolationError, ConvergenceError, empty_host_cache
from .topology import (DistortionReport, ExtremaSet, NeighborScan, SegmentationLabels, compare_plmss,
                       compute_segmentation, compute_segmentation_naive, field_scan, find_extrema, scan_neighbors)
from .correction import (BoundsField, CorrectionConfig, CorrectionResult, DeviceCorrection, EditSet,
                         apply_edit, compute_bounds, iterate_array, run_correction,
                         run_correction_device, validate_error_bound)
from .parallel import (Block, BlockDecomposition, ParallelStats, SyncStrategy, block_domain, decompose,
                       local_converge, run_parallel, sync_ghosts)
from .codec import (FormatError, decode_edits, decode_edits_meta, encode_edits, read_field, read_labels,
                    write_field, write_labels)
from .inputs import (NoiseSpec, PayloadFormatError, PeakSpec, QuantizedPayload, constant, perlin, quantize, ramp,
                     reconstruct, relative_to_absolute)
from .records import (Distortion, DistortionKind, correction_iteration, detect_distortions, extreme_neighbor,
                      is_maximum, is_minimum, propose_corrections)

__version__ = "0.1.0"
