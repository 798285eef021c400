"""B200-native GMP-GR HiPANNS retrieval hot path (drop-in for the reference ``nann``
package's index-build / search / score API on that path).

Host code is Python over the C ABI of ``libgmpgr.so`` (include/gmpgr.h): hand-written
sm_100a kernels for the hop-synchronous C-HiPANNS traversal with fused exact-fp32
metric scoring, the pair scorer, exact brute force and the shard top-k merge.
"""

from .batching import (
    BatchClient,
    BatchEngine,
    BatchQueue,
    Dispatcher,
    DispatchStats,
    EvalRequest,
    GpuBatchEngine,
    ModelBatchEngine,
    run_dispatcher,
)
from .errors import (
    BandError,
    DeviceError,
    FileFormatError,
    InvalidArgumentError,
    NannError,
    NumericError,
    QueueShutdownError,
    WeightOverflowError,
)
from .index import GraphIndex
from .metric import (
    MetricModel,
    Projector,
    RelevanceModel,
    create_model,
    load_model,
    project,
    quantize,
    relevance,
    relevance_batch,
    save_model,
)
from .pool import CandidatePool
from .search import (
    BatchSearchResult,
    SearchParams,
    SearchResult,
    SearchStats,
    brute_force,
    brute_force_batch,
    c_hipanns,
    c_hipanns_batch,
    c_hipanns_scores_batch,
    coverage,
    euclidean_scorer,
    invalidate_device_items,
    model_scorer,
    recall_at,
    table_scorer,
)

__version__ = "0.1.0"

__all__ = [
    "BatchClient", "BatchEngine", "BatchQueue", "BatchSearchResult", "DispatchStats", "Dispatcher",
    "EvalRequest", "ModelBatchEngine", "run_dispatcher", "CandidatePool", "BandError", "DeviceError", "FileFormatError",
    "GpuBatchEngine", "GraphIndex", "InvalidArgumentError", "MetricModel", "NannError",
    "NumericError", "Projector", "QueueShutdownError", "RelevanceModel", "SearchParams",
    "SearchResult", "SearchStats", "WeightOverflowError", "brute_force", "brute_force_batch",
    "c_hipanns", "c_hipanns_batch", "c_hipanns_scores_batch", "coverage", "euclidean_scorer",
    "table_scorer", "create_model", "load_model", "model_scorer",
    "project", "quantize", "recall_at", "relevance", "relevance_batch", "save_model",
    "invalidate_device_items",
]
