// Native control-plane codec: the reference wire format in C++ (host only).
//
// Frame = u32le body_len | u8 kind | body (body_len counts the kind byte);
// integers little-endian fixed width; strings u16 len | utf-8.  Kinds 1..9 =
// Join, Welcome, Announce, Ack, Heartbeat, EpochStart, EpochEnd, Bye,
// Shutdown (reference: pkg/src/batchsocket/wire.py:1-11,77-156,199-341 and the
// facade's codec pkg/frontend/src/sharedloader/abi.py:131-226), plus the two
// extensions of this build: DType code 5 (bf16) and Join v2 (i16 device, u32
// batch_size after the v1 body).  Byte-identical to the Python codec
// (paper_2409_18749_b200/wire.py); tests/test_wire_native.py pins both to
// the golden frames the reference produced.  For non-Python hosts of the
// control plane; the data path never touches it.
#include <cstring>

#include "tsb200.h"

namespace {

constexpr uint32_t MAX_BODY = 65536;
constexpr int MAX_NAME = 255;
constexpr int MAX_NDIM = 8;
const int DTYPE_SIZE[6] = {1, 4, 8, 4, 8, 2};

struct W {
    uint8_t *p;
    size_t cap, n;
    bool ok;
    template <typename T>
    void put(T v) {
        if (n + sizeof(T) > cap) {
            ok = false;
            return;
        }
        memcpy(p + n, &v, sizeof(T));  // little-endian host (x86-64 / aarch64)
        n += sizeof(T);
    }
    void bytes(const void *b, size_t k) {
        if (n + k > cap) {
            ok = false;
            return;
        }
        memcpy(p + n, b, k);
        n += k;
    }
};

struct R {
    const uint8_t *p;
    size_t end, off;
    template <typename T>
    bool get(T &v) {
        if (off + sizeof(T) > end) return false;
        memcpy(&v, p + off, sizeof(T));
        off += sizeof(T);
        return true;
    }
};

int fail(size_t *err_off, size_t off, int code) {
    if (err_off) *err_off = off;
    return code;
}

}  // namespace

extern "C" {

int tsb_wire_encode(const tsb_msg *m, uint8_t *out, size_t cap, size_t *len) {
    if (!m || !out || !len) return TSB_ERR_INVALID;
    W w{out, cap, 0, true};
    w.put<uint32_t>(0);  // body length, patched below
    w.put<uint8_t>(m->kind);
    switch (m->kind) {
        case TSB_MSG_JOIN:
            w.put<uint64_t>(m->consumer_id);
            w.put<uint16_t>(m->protocol_version);
            if (m->protocol_version >= 2) {
                w.put<int16_t>(m->device);
                w.put<uint32_t>(m->batch_size);
            } else if (m->device != -1 || m->batch_size != 0) {
                return TSB_ERR_INVALID;  // v2 fields need protocol_version >= 2
            }
            break;
        case TSB_MSG_WELCOME:
            if (m->epoch_len == 0 || m->admitted > 2) return TSB_ERR_INVALID;
            w.put<uint64_t>(m->consumer_id);
            w.put<uint32_t>(m->epoch);
            w.put<uint64_t>(m->epoch_len);
            w.put<uint64_t>(m->next_batch_index);
            w.put<uint16_t>(m->buffer_depth);
            w.put<uint8_t>(m->admitted);
            break;
        case TSB_MSG_ANNOUNCE: {
            if (m->name_len == 0 || m->name_len > MAX_NAME || m->ndim > MAX_NDIM || m->dtype > 5)
                return TSB_ERR_INVALID;
            uint64_t nb = (uint64_t)DTYPE_SIZE[m->dtype];
            for (int i = 0; i < m->ndim; ++i) nb *= m->shape[i];
            if (nb != m->byte_len) return TSB_ERR_INVALID;
            w.put<uint32_t>(m->epoch);
            w.put<uint64_t>(m->batch_index);
            w.put<uint16_t>(m->name_len);
            w.bytes(m->segment_name, m->name_len);
            w.put<uint64_t>(m->byte_len);
            w.put<uint8_t>(m->dtype);
            w.put<uint8_t>(m->ndim);
            for (int i = 0; i < m->ndim; ++i) w.put<uint64_t>(m->shape[i]);
            w.put<uint32_t>(m->checksum);
            break;
        }
        case TSB_MSG_ACK:
            w.put<uint64_t>(m->consumer_id);
            w.put<uint32_t>(m->epoch);
            w.put<uint64_t>(m->batch_index);
            break;
        case TSB_MSG_HEARTBEAT:
            w.put<uint64_t>(m->consumer_id);
            w.put<uint64_t>(m->monotonic_millis);
            break;
        case TSB_MSG_EPOCH_START:
            if (m->epoch_len == 0) return TSB_ERR_INVALID;
            w.put<uint32_t>(m->epoch);
            w.put<uint64_t>(m->epoch_len);
            break;
        case TSB_MSG_EPOCH_END:
            w.put<uint32_t>(m->epoch);
            break;
        case TSB_MSG_BYE:
            w.put<uint64_t>(m->consumer_id);
            break;
        case TSB_MSG_SHUTDOWN:
            break;
        default:
            return TSB_ERR_INVALID;
    }
    if (!w.ok) return TSB_ERR_INVALID;
    const uint32_t body = (uint32_t)(w.n - 4);
    memcpy(out, &body, 4);
    *len = w.n;
    return TSB_OK;
}

int tsb_wire_decode(const uint8_t *frame, size_t len, tsb_msg *m, size_t *err_off) {
    if (!frame || !m) return TSB_ERR_INVALID;
    memset(m, 0, sizeof(*m));
    m->device = -1;
    if (len < 4) return fail(err_off, 0, TSB_ERR_CORRUPT);
    uint32_t body = 0;
    memcpy(&body, frame, 4);
    if (body == 0) return fail(err_off, 4, TSB_ERR_CORRUPT);
    if (body > MAX_BODY) return fail(err_off, 0, TSB_ERR_CORRUPT);
    if (len != 4 + (size_t)body) return fail(err_off, 4, TSB_ERR_CORRUPT);
    R r{frame, len, 5};
    m->kind = frame[4];
    bool ok = true;
    switch (m->kind) {
        case TSB_MSG_JOIN:
            ok = r.get(m->consumer_id) && r.get(m->protocol_version);
            if (ok && body - 1 == 16) {  // Join v2
                if (m->protocol_version < 2) return fail(err_off, 13, TSB_ERR_CORRUPT);
                ok = r.get(m->device) && r.get(m->batch_size);
            }
            break;
        case TSB_MSG_WELCOME:
            ok = r.get(m->consumer_id) && r.get(m->epoch) && r.get(m->epoch_len) &&
                 r.get(m->next_batch_index) && r.get(m->buffer_depth) && r.get(m->admitted);
            if (ok && m->epoch_len == 0) return fail(err_off, 13, TSB_ERR_CORRUPT);
            if (ok && m->admitted > 2) return fail(err_off, r.off - 1, TSB_ERR_CORRUPT);
            break;
        case TSB_MSG_ANNOUNCE: {
            ok = r.get(m->epoch) && r.get(m->batch_index) && r.get(m->name_len);
            if (!ok) break;
            if (m->name_len > MAX_NAME) return fail(err_off, r.off - 2, TSB_ERR_CORRUPT);
            if (r.off + m->name_len > r.end) return fail(err_off, r.off, TSB_ERR_CORRUPT);
            memcpy(m->segment_name, frame + r.off, m->name_len);
            m->segment_name[m->name_len] = 0;
            r.off += m->name_len;
            ok = r.get(m->byte_len) && r.get(m->dtype) && r.get(m->ndim);
            if (!ok) break;
            if (m->ndim > MAX_NDIM) return fail(err_off, r.off - 1, TSB_ERR_CORRUPT);
            for (int i = 0; ok && i < m->ndim; ++i) ok = r.get(m->shape[i]);
            ok = ok && r.get(m->checksum);
            if (!ok) break;
            if (m->dtype > 5) return fail(err_off, r.off - 8 * m->ndim - 6, TSB_ERR_CORRUPT);
            uint64_t nb = (uint64_t)DTYPE_SIZE[m->dtype];
            for (int i = 0; i < m->ndim; ++i) nb *= m->shape[i];
            if (nb != m->byte_len || m->name_len == 0) return fail(err_off, 5, TSB_ERR_CORRUPT);
            break;
        }
        case TSB_MSG_ACK:
            ok = r.get(m->consumer_id) && r.get(m->epoch) && r.get(m->batch_index);
            break;
        case TSB_MSG_HEARTBEAT:
            ok = r.get(m->consumer_id) && r.get(m->monotonic_millis);
            break;
        case TSB_MSG_EPOCH_START:
            ok = r.get(m->epoch) && r.get(m->epoch_len);
            if (ok && m->epoch_len == 0) return fail(err_off, 9, TSB_ERR_CORRUPT);
            break;
        case TSB_MSG_EPOCH_END:
            ok = r.get(m->epoch);
            break;
        case TSB_MSG_BYE:
            ok = r.get(m->consumer_id);
            break;
        case TSB_MSG_SHUTDOWN:
            break;
        default:
            return fail(err_off, 4, TSB_ERR_CORRUPT);
    }
    if (!ok) return fail(err_off, r.off, TSB_ERR_CORRUPT);
    if (r.off != r.end) return fail(err_off, r.off, TSB_ERR_CORRUPT);  // trailing bytes
    return TSB_OK;
}

}  // extern "C"
