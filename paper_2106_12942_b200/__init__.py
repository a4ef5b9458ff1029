"""B200-native RHSEG: recursive hierarchical segmentation of hyperspectral
cubes (arXiv 2106.12942 / the `rhseg` reference package), hot path on sm_100a.

Drop-in entry points (same names, arguments and results as the reference):
  hseg_run / hseg_step / search_table / scan_adjacent / scan_nonadjacent  (engine)
  rhseg_run / B200Executor.execute -> RhsegResult                          (recursive)
"""

from .dissim import MEASURES, acos_fdlibm, euclidean, resolve_measure, sam, sqrt_bsmse
from .engine import (
    BestPairTable,
    GraphSnapshot,
    HsegParams,
    PerPair,
    PerRegion,
    ProfileStats,
    Sequential,
    best_adjacent_pair,
    best_nonadjacent_pair,
    hseg_run,
    hseg_step,
    make_strategy,
    reduce_best,
    scan_adjacent,
    scan_nonadjacent,
    search_table,
    snapshot,
)
from .errors import (
    BandMismatch,
    DeadRegion,
    DeviceError,
    DimensionMismatch,
    ExtensionMissing,
    IndivisibleImage,
    InfeasibleLayout,
    LevelOutOfRange,
    RhsegError,
    SelfMerge,
    ShapeMismatch,
    TooManyLabels,
)
from .graph import (
    LabelMap,
    MergeHierarchy,
    MergeKind,
    MergeRecord,
    Region,
    RegionGraph,
    dense_renumber,
    extract_labels,
    init_from_presegmentation,
    init_region_graph,
    label_map_from_graph,
    merge_regions,
)
from .image import HyperImage
from .recursive import (
    B200Executor,
    RecordList,
    RhsegParams,
    RhsegResult,
    assemble_result,
    rhseg_run,
    run_leaf,
    run_upper_levels,
)
from .sections import SectionId, SectionTask, log_order, partition, section_side, stitch, total_sections
from .synth import GroundTruth, gen_synthetic

__version__ = "0.1.0"
