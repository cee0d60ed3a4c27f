"""Debug harness: heterogeneous consumers on one producer; dumps ring control
words and consumer state if the pipeline stalls."""
import sys
import threading
import time

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import torch  # noqa: E402

import test_gpu_facade_multi as T  # noqa: E402
from paper_2409_18749_b200 import SharedLoader, TensorProducer  # noqa: E402

N, B = 128, 32
ld = T._loader(N, B, "float32", seed=5)
sizes = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "8,16,32,64,24").split(",")]
b_, a_ = "unix:/tmp/dbg_b.sock", "unix:/tmp/dbg_a.sock"
producer = TensorProducer(ld, broadcast=b_, aggregate=a_, heartbeat_timeout_s=60.0,
                          min_consumers=len(sizes), ring_slots=4)


def run():
    for _ in range(2):
        for _ in producer:
            pass
    producer.join(30)


pt = threading.Thread(target=run, daemon=True)
pt.start()
loaders = [SharedLoader(b_, a_, consumer_id=100 + i, batch_size=b) for i, b in enumerate(sizes)]
outs = [[] for _ in sizes]
ts = [threading.Thread(target=T._consume, args=(ld_, 2, outs[i]), daemon=True)
      for i, ld_ in enumerate(loaders)]
for t in ts:
    t.start()
t0 = time.time()
while any(t.is_alive() for t in ts) and time.time() - t0 < 20:
    time.sleep(0.5)
if any(t.is_alive() for t in ts):
    r = producer.ring
    print("STALL ready:", [r.read_ready(s) for s in range(r.slots)])
    print("cursors:", [r.read_cursor(c) for c in range(6)], "ret", r.read_cursor(producer._max_consumers))
    print("stats", producer.stats, "epoch", producer._epoch, "announced_in_epoch", producer._announced_in_epoch)
    for b, L_ in zip(sizes, loaders):
        print("b", b, "fetched", L_.fetched, "released", L_._released, "q", len(L_._queue),
              [x if isinstance(x, str) else (x.epoch, x.batch_index) for x in L_._queue][:6],
              "next_index", L_._next_index, "cur_epoch", L_._current_epoch, "waiting", L_._waiting,
              "cursor_idx", L_._cursor)
    sys.stdout.flush()
for t in ts:
    t.join(60)
for b, got in zip(sizes, outs):
    print("b", b, [len(e) if not isinstance(e, str) else e[-300:] for e in got])
print(producer.drops)
