// Native control-plane hub: the producer's per-batch socket work off the GIL.
//
// The reference producer runs one reader thread per consumer connection and
// a coordinator that broadcasts each Announce over every consumer socket
// (bs/producer.py:379-438, bs/transport.py:94-146).  In a Python producer
// that per-consumer, per-batch work -- decoding every wire Ack and writing
// every Announce -- serialises on the interpreter lock and grows linearly
// with the consumer count (profiles/r1: ~18 us per consumer per batch).
// The hub moves it to native code:
//   * one epoll thread reads every admitted consumer's aggregate socket,
//     decodes frames with the native codec (tsb_wire.cpp) and queues Ack /
//     Heartbeat / Bye / closed events, which the producer drains in one call;
//   * tsb_hub_broadcast writes one encoded frame to many sockets in one call.
// Join / Welcome and the rest of the handshake stay in Python; a consumer's
// aggregate socket is handed to the hub once admitted (with any bytes the
// Python reader had already buffered).
#include <errno.h>
#include <sys/epoll.h>
#include <sys/eventfd.h>
#include <sys/socket.h>
#include <time.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <vector>

#include "tsb200.h"

namespace tsb {
void set_error(const char *fmt, ...);
}

namespace {
int64_t now_us() {
    struct timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return (int64_t)t.tv_sec * 1000000 + t.tv_nsec / 1000;
}
struct HubConn {
    std::vector<uint8_t> buf;
    uint64_t consumer_id;
};
}  // namespace

struct tsb_hub {
    int epfd = -1;
    int wake = -1;
    std::thread th;
    std::atomic<bool> stop{false};
    std::mutex mu;                      // guards conns, events and acked
    std::condition_variable cv;         // an Ack raised some consumer's acked seq
    std::unordered_map<int, HubConn> conns;
    std::vector<tsb_hub_event> events;
    uint64_t epoch_len = 0;             // 0: acked seqs are not tracked
    std::unordered_map<uint64_t, uint64_t> acked;  // consumer id -> highest acked seq
    uint64_t drift_max = 0;             // max - min acked over registered consumers, any Ack

    void sample_drift() {  // caller holds mu
        uint64_t lo = ~0ull, hi = 0;
        for (const auto &kv : acked) {
            if (kv.second >= (1ull << 61)) continue;  // departed (sentinel)
            if (kv.second < lo) lo = kv.second;
            if (kv.second > hi) hi = kv.second;
        }
        if (hi >= lo && hi - lo > drift_max) drift_max = hi - lo;
    }

    bool all_acked(const uint64_t *ids, int n, uint64_t need) const {  // caller holds mu
        for (int i = 0; i < n; ++i) {
            auto it = acked.find(ids[i]);
            if (it == acked.end() || it->second < need) return false;
        }
        return true;
    }

    void push(uint8_t kind, uint64_t cid, uint32_t epoch, uint64_t bi, int fd) {
        tsb_hub_event e{};
        e.kind = kind;
        e.consumer_id = cid;
        e.epoch = epoch;
        e.batch_index = bi;
        e.t_us = now_us();
        e.fd = fd;
        events.push_back(e);
    }

    void close_fd(int fd) {  // caller holds mu
        epoll_ctl(epfd, EPOLL_CTL_DEL, fd, nullptr);
        auto it = conns.find(fd);
        const uint64_t cid = it == conns.end() ? 0 : it->second.consumer_id;
        conns.erase(fd);
        push(0, cid, 0, 0, fd);  // kind 0: connection closed / protocol error
    }

    // parse every complete frame in c.buf; false on a protocol error
    bool parse(int fd, HubConn &c) {
        size_t off = 0;
        while (c.buf.size() - off >= 4) {
            uint32_t body = 0;
            memcpy(&body, c.buf.data() + off, 4);
            if (body == 0 || body > 65536) return false;
            if (c.buf.size() - off < 4 + (size_t)body) break;
            tsb_msg m;
            size_t eo = 0;
            if (tsb_wire_decode(c.buf.data() + off, 4 + body, &m, &eo) != TSB_OK) return false;
            if (m.kind == TSB_MSG_ACK || m.kind == TSB_MSG_HEARTBEAT || m.kind == TSB_MSG_BYE)
                push(m.kind, m.consumer_id, m.epoch, m.batch_index, fd);
            if (m.kind == TSB_MSG_ACK && epoch_len) {
                // max-monotone, as the reference's ack cursor (bs/producer.py:251)
                const uint64_t seq = (uint64_t)m.epoch * epoch_len + m.batch_index + 1;
                auto it = acked.find(m.consumer_id);
                if (it != acked.end() && seq > it->second) {
                    it->second = seq;
                    sample_drift();
                    cv.notify_all();
                }
            }
            off += 4 + body;
        }
        c.buf.erase(c.buf.begin(), c.buf.begin() + off);
        return true;
    }

    void loop() {
        epoll_event evs[64];
        std::vector<uint8_t> tmp(65536);
        while (!stop.load(std::memory_order_acquire)) {
            const int n = epoll_wait(epfd, evs, 64, 200);
            for (int i = 0; i < n; ++i) {
                const int fd = evs[i].data.fd;
                if (fd == wake) {
                    uint64_t v;
                    if (read(wake, &v, sizeof v) < 0) { /* drained */ }
                    continue;
                }
                const ssize_t r = recv(fd, tmp.data(), tmp.size(), MSG_DONTWAIT);
                std::lock_guard<std::mutex> lk(mu);
                auto it = conns.find(fd);
                if (it == conns.end()) continue;  // removed meanwhile
                if (r > 0) {
                    it->second.buf.insert(it->second.buf.end(), tmp.data(), tmp.data() + r);
                    if (!parse(fd, it->second)) close_fd(fd);
                } else if (r == 0 || (errno != EAGAIN && errno != EWOULDBLOCK && errno != EINTR)) {
                    close_fd(fd);
                }
            }
        }
    }
};

extern "C" {

int tsb_hub_create(tsb_hub **out) {
    if (!out) return TSB_ERR_INVALID;
    tsb_hub *h = new tsb_hub{};
    h->epfd = epoll_create1(EPOLL_CLOEXEC);
    h->wake = eventfd(0, EFD_NONBLOCK | EFD_CLOEXEC);
    if (h->epfd < 0 || h->wake < 0) {
        tsb::set_error("hub: epoll/eventfd: %s", strerror(errno));
        if (h->epfd >= 0) close(h->epfd);
        if (h->wake >= 0) close(h->wake);
        delete h;
        return TSB_ERR_INVALID;
    }
    epoll_event ev{};
    ev.events = EPOLLIN;
    ev.data.fd = h->wake;
    epoll_ctl(h->epfd, EPOLL_CTL_ADD, h->wake, &ev);
    h->th = std::thread([h] { h->loop(); });
    *out = h;
    return TSB_OK;
}

int tsb_hub_add(tsb_hub *h, int fd, uint64_t consumer_id, const uint8_t *pending, size_t n) {
    if (!h || fd < 0) return TSB_ERR_INVALID;
    std::lock_guard<std::mutex> lk(h->mu);
    HubConn &c = h->conns[fd];
    c.consumer_id = consumer_id;
    c.buf.assign(pending, pending + (pending ? n : 0));
    if (!h->parse(fd, c)) {
        h->close_fd(fd);
        return TSB_OK;
    }
    epoll_event ev{};
    ev.events = EPOLLIN | EPOLLRDHUP;
    ev.data.fd = fd;
    if (epoll_ctl(h->epfd, EPOLL_CTL_ADD, fd, &ev) != 0) {
        tsb::set_error("hub: epoll_ctl(ADD, %d): %s", fd, strerror(errno));
        h->conns.erase(fd);
        return TSB_ERR_INVALID;
    }
    return TSB_OK;
}

int tsb_hub_remove(tsb_hub *h, int fd) {
    if (!h) return TSB_ERR_INVALID;
    std::lock_guard<std::mutex> lk(h->mu);
    epoll_ctl(h->epfd, EPOLL_CTL_DEL, fd, nullptr);
    h->conns.erase(fd);
    return TSB_OK;
}

int tsb_hub_drain(tsb_hub *h, tsb_hub_event *out, int cap, int *n) {
    if (!h || !out || !n || cap < 0) return TSB_ERR_INVALID;
    std::lock_guard<std::mutex> lk(h->mu);
    const int k = (int)h->events.size() < cap ? (int)h->events.size() : cap;
    memcpy(out, h->events.data(), sizeof(tsb_hub_event) * (size_t)k);
    h->events.erase(h->events.begin(), h->events.begin() + k);
    *n = k;
    return TSB_OK;
}

int tsb_hub_broadcast(const int *fds, int n, const uint8_t *frame, size_t len, int *failed) {
    if ((!fds && n) || !frame) return TSB_ERR_INVALID;
    for (int i = 0; i < n; ++i) {
        size_t off = 0;
        int bad = 0;
        while (off < len) {
            const ssize_t w = send(fds[i], frame + off, len - off, MSG_NOSIGNAL);
            if (w < 0) {
                if (errno == EINTR) continue;
                bad = 1;
                break;
            }
            off += (size_t)w;
        }
        if (failed) failed[i] = bad;
    }
    return TSB_OK;
}

int tsb_hub_set_epoch_len(tsb_hub *h, uint64_t epoch_len) {
    if (!h) return TSB_ERR_INVALID;
    std::lock_guard<std::mutex> lk(h->mu);
    h->epoch_len = epoch_len;
    return TSB_OK;
}

int tsb_hub_set_acked(tsb_hub *h, uint64_t consumer_id, uint64_t seq) {
    if (!h) return TSB_ERR_INVALID;
    std::lock_guard<std::mutex> lk(h->mu);
    h->acked[consumer_id] = seq;
    h->cv.notify_all();
    return TSB_OK;
}

int tsb_hub_read_acked(tsb_hub *h, uint64_t consumer_id, uint64_t *seq) {
    if (!h || !seq) return TSB_ERR_INVALID;
    std::lock_guard<std::mutex> lk(h->mu);
    auto it = h->acked.find(consumer_id);
    *seq = it == h->acked.end() ? 0 : it->second;
    return TSB_OK;
}

int tsb_hub_wait_acked(tsb_hub *h, const uint64_t *consumer_ids, int n, uint64_t need,
                       int64_t timeout_us) {
    if (!h || (n && !consumer_ids) || n < 0) return TSB_ERR_INVALID;
    std::unique_lock<std::mutex> lk(h->mu);
    auto ok = [&] { return h->all_acked(consumer_ids, n, need); };
    if (timeout_us < 0) {
        h->cv.wait(lk, ok);
        return TSB_OK;
    }
    return h->cv.wait_for(lk, std::chrono::microseconds(timeout_us), ok) ? TSB_OK
                                                                        : TSB_ERR_STALE;
}

int tsb_hub_drift_max(tsb_hub *h, uint64_t *drift) {
    if (!h || !drift) return TSB_ERR_INVALID;
    std::lock_guard<std::mutex> lk(h->mu);
    *drift = h->drift_max;
    return TSB_OK;
}

int tsb_hub_destroy(tsb_hub *h) {
    if (!h) return TSB_OK;
    h->stop.store(true, std::memory_order_release);
    uint64_t one = 1;
    if (write(h->wake, &one, sizeof one) < 0) { /* the 200 ms epoll timeout still ends the loop */ }
    if (h->th.joinable()) h->th.join();
    close(h->epfd);
    close(h->wake);
    delete h;
    return TSB_OK;
}

}  // extern "C"
