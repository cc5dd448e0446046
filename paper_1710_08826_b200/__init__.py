"""B200-native engine for the GooFit 2.0 hot path, plugged into the reference.

The reference (parafit: ``Variable``, ``PdfNode`` builders, ``UnbinnedDataSet``,
``nll``, ``FitManager``, ``shard``/``reduce_partials``) stays the API; this
package supplies what runs beneath it on the GPU (hand-written sm_100a CUDA in
libpfb200.so, reached through a C ABI):

* :class:`DeviceBackend` -- the reference ``Backend`` protocol
  (P/engine.py:32-97): the reference's own ``nll`` and ``FitManager`` run every
  NLL as one fused kernel launch with an exact reduction;
* :mod:`.norms` -- device normalisation integrals registered through the
  reference's ``register_cached_norm`` (Gauss-Legendre quadrature, Dalitz
  overlap integrals), recomputed only when the reference cache says so;
* :class:`DeviceDataSet` -- a reference ``UnbinnedDataSet`` with an HBM copy;
* :class:`DeviceFitManager` -- the reference ``FitManager`` with batched
  finite-difference / Hesse stencils;
* :mod:`.sharding` -- device partials for the reference's shard/reduce and one
  process per GPU (:class:`ShardedNll`);
* :mod:`.mcgen`, :mod:`.dataio` -- the reference's toy generators and binary
  ingest straight into HBM.

There is no CPU fallback: the product imports libpfb200.so or fails
(``_lib.NativeMissing``), and a context without a GPU fails with
``PFB_E_NO_DEVICE``.
"""

from . import _reference
from ._reference import parafit
from .datasets import DeviceDataSet, as_device_dataset, bin_fill, binned_nll
from .engine import DeviceBackend, DeviceContext, default_backend, device_context, nll, nll_block_sums, shard_bounds
from .fitting import DeviceFitManager, fit_manager_run
from .norms import device_norms, install, quadrature, reference_norms, uninstall
from .sharding import ShardedNll, components_from_acc, partial_nll, sharded_nll

__version__ = "0.2.0"

__all__ = [
    "DeviceBackend", "DeviceContext", "DeviceDataSet", "DeviceFitManager", "ShardedNll", "as_device_dataset",
    "bin_fill", "binned_nll", "components_from_acc", "default_backend", "device_context", "device_norms",
    "fit_manager_run", "install", "nll", "nll_block_sums", "parafit", "partial_nll", "quadrature",
    "reference_norms", "shard_bounds", "sharded_nll", "uninstall",
]
