"""B200-native drop-in for the row-partitioned GCN training path of `gcnpart`
(arXiv 2212.05009): partition → communication plan → scatter → train epochs,
with every per-epoch operation (SpMM, dense transforms, halo pack/exchange,
loss, ΔW reduction, SGD) running as hand-written sm_100a kernels in
`lib/libgcnb.so` (C ABI: include/gcnb.h).

The names below are the reference's public API for this path
(gcnpart/__init__.py:7-67); host-side types accept gcnpart's own objects by
duck typing.  Partitioners other than RP and the reporting/CLI layers are
outside this package's scope.
"""

from ._lib import CommError
from .comm import CommPlan, PlanVolume, build_comm_plan, plan_volume
from .host import (
    BalanceInfeasibleError,
    GcnModel,
    LabelSet,
    MiniBatchSpec,
    Partition,
    PartitionConfig,
    induced_pattern,
    init_model,
    random_partition,
    sample_batches,
)
from .runtime import (
    DeviceNetwork,
    EpochMetrics,
    FullBatch,
    MessageRecord,
    MiniBatch,
    ProcState,
    SimNetwork,
    allreduce_sum,
    parallel_backprop,
    parallel_feedforward,
    scatter,
    train_epochs,
)
from .sparse import CsrMatrix, RowBlock, gather_rows, normalize_adjacency, spmm, transpose_sparse

__all__ = [n for n in dir() if not n.startswith("_")]
__version__ = "0.1.0"
