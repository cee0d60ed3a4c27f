"""Host control plane: framed stream sockets (unix:/path or tcp:host:port).

Same endpoint syntax and env fallbacks as the reference (bs/transport.py:27-146,
sl/config.py:7-34).  Frames are tiny; the data plane never touches sockets.
"""

from __future__ import annotations

import os
import socket
import threading
import time

from . import wire

ENV_BROADCAST = "BATCHSOCKET_BROADCAST"
ENV_AGGREGATE = "BATCHSOCKET_AGGREGATE"


def endpoints_from_env(broadcast: str | None, aggregate: str | None) -> tuple[str, str]:
    broadcast = broadcast or os.environ.get(ENV_BROADCAST)
    aggregate = aggregate or os.environ.get(ENV_AGGREGATE)
    if not broadcast or not aggregate:
        raise ValueError("endpoints required: pass broadcast=/aggregate= or set "
                         f"{ENV_BROADCAST} and {ENV_AGGREGATE}")
    return broadcast, aggregate


def parse_endpoint(spec: str):
    spec = spec.strip()
    if spec.startswith("unix:"):
        return "unix", spec[5:]
    if spec.startswith("tcp:"):
        host, _, port = spec[4:].rpartition(":")
        return "tcp", (host, int(port))
    if "/" in spec:
        return "unix", spec
    host, sep, port = spec.rpartition(":")
    if sep and port.isdigit():
        return "tcp", (host, int(port))
    raise ValueError(f"cannot parse endpoint {spec!r}")


def listen(endpoint: str) -> socket.socket:
    fam, addr = parse_endpoint(endpoint)
    if fam == "unix":
        s = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        try:
            os.unlink(addr)
        except FileNotFoundError:
            pass
    else:
        s = socket.socket(socket.AF_INET, socket.SOCK_STREAM)
        s.setsockopt(socket.SOL_SOCKET, socket.SO_REUSEADDR, 1)
    s.bind(addr)
    s.listen(64)
    return s


def dial(endpoint: str, timeout: float) -> socket.socket:
    from .errors import StreamError

    fam, addr = parse_endpoint(endpoint)
    deadline = time.monotonic() + timeout
    while True:
        s = socket.socket(socket.AF_UNIX if fam == "unix" else socket.AF_INET, socket.SOCK_STREAM)
        try:
            s.settimeout(2.0)
            s.connect(addr)
            s.settimeout(None)
            if fam == "tcp":
                s.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)
            return s
        except OSError as exc:
            s.close()
            if time.monotonic() > deadline:
                raise StreamError(f"cannot reach producer at {endpoint}: {exc}") from exc
            time.sleep(0.02)


HANDOFF = object()  # on_msg return value: stop the Python reader, hand the socket off


class Conn:
    """A socket with a send lock and a frame reader thread."""

    def __init__(self, sock: socket.socket):
        self.sock = sock
        self._lock = threading.Lock()
        self.closed = False

    def send(self, msg) -> None:
        self.send_raw(wire.encode(msg))

    def send_raw(self, data: bytes) -> None:
        with self._lock:
            self.sock.sendall(data)

    def start_reader(self, on_msg, on_close, name: str = "reader",
                     on_handoff=None) -> threading.Thread:
        """Read frames on a thread.  If on_msg returns ``HANDOFF`` the thread
        stops reading (the socket stays open) and ``on_handoff(pending_bytes)``
        gets what was already read past that frame -- used to pass an admitted
        consumer's socket to the native hub."""

        def run():
            dec = wire.FrameDecoder()
            try:
                while True:
                    data = self.sock.recv(65536)
                    if not data:
                        break
                    msgs = dec.feed(data)
                    for i, m in enumerate(msgs):
                        if on_msg(m) is HANDOFF and on_handoff is not None:
                            rest = b"".join(wire.encode(x) for x in msgs[i + 1:])
                            on_handoff(rest + dec.take_pending())
                            return
            except (OSError, ValueError):
                pass
            on_close()

        t = threading.Thread(target=run, name=name, daemon=True)
        t.start()
        return t

    def close(self) -> None:
        if not self.closed:
            self.closed = True
            try:
                self.sock.shutdown(socket.SHUT_RDWR)
            except OSError:
                pass
            try:
                self.sock.close()
            except OSError:
                pass


def mono_ms() -> int:
    return int(time.monotonic() * 1000)
