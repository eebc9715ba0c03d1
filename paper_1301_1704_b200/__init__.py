"""paper_1301_1704_b200 — B200-native (sm_100a) FMM data-structure build.

Drop-in for the `fmmkit` build path (Hu, Gumerov & Duraiswami, arXiv
1301.1704, Alg. 1-5): `build_all`, `sort_points` and the sub-builders keep the
reference's names, arguments, errors and output layout
(pkg/src/fmmkit/lists.py, pseudosort.py); `kernels` is a drop-in for the
`fmmkit.backend.kernels` plugin (pkg/src/fmmkit/backend.py).  All compute is
hand-written CUDA in libfmmb200.so behind the C ABI in include/fmmb200.h.
"""

from .errors import (
    CapacityError,
    DomainError,
    FmmError,
    InfeasiblePartitionError,
    NativeError,
    RoutingError,
)
from .lists import (
    FmmStructures,
    LevelDirectory,
    NeighborTable,
    TranslationStencils,
    build_all,
    build_all_device,
    build_level_directory,
    build_neighbor_table,
    build_translation_stencils,
    dump_structures,
    gather_adjacent_sources,
    load_structures,
    propagate_to_parents,
)
from . import container
from .boxtype import BoxType, TypedBoxList, classify
from .partition import PartitionPlan, choose_partition
from .scan import compact_flags, exclusive_scan
from .fmm import direct_sum, near_field_potentials
from .pseudosort import (
    DEFAULT_HISTOGRAM_BUDGET,
    MAX_LEVEL,
    SortedPointSet,
    build_bookmarks,
    choose_max_level,
    histogram_and_sort_index,
    reorder,
    sort_points,
    sort_points_device,
)

__all__ = [name for name in dir() if not name.startswith("_")]
