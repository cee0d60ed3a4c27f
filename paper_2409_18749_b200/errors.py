"""Exception classes mirroring the reference (payload.py:48-61, wire.py:33-46,
sl/loader.py:23-24, sl/producer.py:29-30)."""


class PayloadError(Exception):
    pass


class StaleHandleError(PayloadError):
    """The slot/handle no longer exists (released before this map)."""


class CorruptSegmentError(PayloadError):
    """Slot failed magic/version/size/checksum validation."""


class ResourceError(PayloadError):
    """Device memory / CUDA resources could not be allocated."""


class DeviceError(PayloadError):
    """Operation not supported on this device/driver."""


class LibraryMissing(RuntimeError):
    """libtsb200.so is not built or cannot be loaded: there is no CPU fallback."""


class StreamError(RuntimeError):
    """Connection to the producer was lost mid-stream (sl/loader.py:23-24)."""


class ProducerClosed(RuntimeError):
    """join() was already called (sl/producer.py:29-30)."""


class ProtocolError(Exception):
    """Peer violated the wire protocol (bs/consumer.py)."""
