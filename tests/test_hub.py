"""Native control-plane hub on CPU (socketpairs): frames handed over with a
reader's leftover bytes, Ack/Heartbeat/Bye decoded natively, closure events,
and one-call broadcast of a frame to many sockets."""

import socket
import time

from paper_2409_18749_b200.hub import Hub
from paper_2409_18749_b200.wire import Ack, Announce, Bye, FrameDecoder, Heartbeat, encode


def wait_events(hub, n, timeout=5.0):
    out, t0 = [], time.time()
    while len(out) < n and time.time() - t0 < timeout:
        out += hub.drain()
        time.sleep(0.005)
    return out


def test_hub_reads_acks_heartbeats_bye_and_closure():
    hub = Hub()
    a, b = socket.socketpair()
    pending = encode(Ack(7, 0, 1))  # bytes a Python reader had already buffered
    hub.add(a.fileno(), 7, pending)
    b.sendall(encode(Ack(7, 0, 2)) + encode(Heartbeat(7, 123)))
    b.sendall(encode(Ack(7, 1, 0))[:10])  # split frame
    time.sleep(0.05)
    b.sendall(encode(Ack(7, 1, 0))[10:] + encode(Bye(7)))
    ev = wait_events(hub, 5)
    assert [(k, c, e, i) for k, c, e, i, _, _ in ev] == [
        (4, 7, 0, 1), (4, 7, 0, 2), (5, 7, 0, 0), (4, 7, 1, 0), (8, 7, 0, 0)]
    assert all(fd == a.fileno() for *_, fd in ev)
    b.close()
    ev = wait_events(hub, 1)
    assert ev and ev[0][0] == 0 and ev[0][5] == a.fileno()
    hub.close()
    a.close()


def test_hub_protocol_error_closes():
    hub = Hub()
    a, b = socket.socketpair()
    hub.add(a.fileno(), 3)
    b.sendall(b"\x00\x00\x00\x00")  # zero-length body
    ev = wait_events(hub, 1)
    assert ev and ev[0][0] == 0
    hub.remove(a.fileno())
    hub.close()
    a.close()
    b.close()


def test_broadcast_one_frame_to_many_sockets():
    pairs = [socket.socketpair() for _ in range(5)]
    frame = encode(Announce(0, 3, "tsb1:ab:1:xyz", 4, 0, (4,), 0))
    assert Hub.broadcast([p[0].fileno() for p in pairs], frame) == []
    for _, r in pairs:
        assert FrameDecoder().feed(r.recv(4096)) == [Announce(0, 3, "tsb1:ab:1:xyz", 4, 0, (4,), 0)]
    pairs[2][1].close()
    failed = Hub.broadcast([p[0].fileno() for p in pairs], frame)
    assert failed == [pairs[2][0].fileno()]
    for s, r in pairs:
        s.close()
        r.close()
