"""B200-native NLL engine for the GooFit 2.0 hot path (reference: parafit).

Public surface mirrors the reference package's names for this path:
Variable / set_value / snapshot / UnbinnedDataSet (core), gaussian /
exponential / polynomial / add_pdf / prod_pdf (pdf), DecayChannel /
ResonanceTerm / dalitz_pdf / compute_integrals / dalitz_norm (dalitz),
NormalizationStore / resolve_norms / nll / binned_nll (engine), BinnedDataSet
(core), shard / partial_nll /
reduce_partials / sharded_nll (sharding) -- plus :class:`DeviceBackend`, a
drop-in ``Backend`` for the reference's own ``nll`` / ``FitManager``.

Evaluation runs only in libpfb200.so (hand-written sm_100a CUDA); there is no
CPU fallback.
"""

from .core import (
    BinnedDataSet,
    ParameterRegistry,
    ParameterSnapshot,
    UnbinnedDataSet,
    Variable,
    set_value,
    snapshot,
)
from .dalitz import (
    DecayChannel,
    IntegralCache,
    ResonanceTerm,
    compute_integrals,
    dalitz_norm,
    dalitz_pdf,
    integration_grid,
)
from .engine import (
    DeviceBackend,
    NormalizationStore,
    binned_nll,
    cached_norm,
    device_context,
    nll,
    nll_block_sums,
    register_cached_norm,
    resolve_norms,
)
from .errors import ParafitError
from .pdf import NormalizationValue, PdfNode, add_pdf, exponential, gaussian, normalize, polynomial, prod_pdf
from .sharding import PartialSum, Shard, ShardedNll, partial_nll, reduce_partials, shard, shard_bounds, sharded_nll

__version__ = "0.1.0"

__all__ = [
    "BinnedDataSet", "binned_nll", "DecayChannel", "DeviceBackend", "IntegralCache", "NormalizationStore", "NormalizationValue",
    "ParafitError", "ParameterRegistry", "ParameterSnapshot", "PartialSum", "PdfNode", "ResonanceTerm",
    "Shard", "ShardedNll", "UnbinnedDataSet", "Variable", "add_pdf", "cached_norm", "compute_integrals",
    "dalitz_norm", "dalitz_pdf", "device_context", "exponential", "gaussian", "integration_grid", "nll",
    "nll_block_sums", "normalize", "partial_nll", "polynomial", "prod_pdf", "reduce_partials",
    "register_cached_norm", "resolve_norms", "set_value", "shard", "shard_bounds", "sharded_nll", "snapshot",
]
