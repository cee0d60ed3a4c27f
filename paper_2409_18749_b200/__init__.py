"""B200-native shared-loading data plane (TensorSocket, arXiv 2409.18749).

Drop-in for the reference's facade (``sharedloader``: ``TensorProducer``,
``SharedLoader``) with ``TensorConsumer`` as the paper's name for the
consumer.  Batches live in a device-HBM ring; collate/augment, CRC, fan-out
and rebatch are hand-written sm_100a kernels in ``libtsb200.so`` (C ABI:
``include/tsb200.h``).  There is no CPU fallback.
"""

from .errors import (CorruptSegmentError, DeviceError, LibraryMissing, PayloadError,  # noqa: F401
                     ProducerClosed, ProtocolError, ResourceError, StaleHandleError, StreamError)

__version__ = "0.1.0"


def __getattr__(name):
    # lazy: importing the package must not require a GPU
    if name in ("TensorProducer",):
        from .producer import TensorProducer

        return TensorProducer
    if name in ("SharedLoader", "TensorConsumer"):
        from . import loader

        return getattr(loader, name)
    if name in ("DeviceRing",):
        from .ring import DeviceRing

        return DeviceRing
    if name in ("CollateLoader", "StoreSource", "SyntheticSource", "DatasetSpec", "AugmentSpec",
                "JpegSource"):
        from . import collate

        return getattr(collate, name)
    raise AttributeError(name)
