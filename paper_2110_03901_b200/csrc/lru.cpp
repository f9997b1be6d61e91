// lru.cpp -- host-side LRU replay behind blocksched.reuse_traffic.
//
// The reference evaluates its subtile orders with a fully-associative LRU
// over gathered element keys (_native.pyx:102-149, blocksched.py:131-151).
// That is an inherently sequential analysis model, not device work, so it
// stays on the host in C++: a flat open-addressing index (key -> slot) plus
// an intrusive recency list, O(1) per access, no per-access allocation.
#include <cstdint>
#include <vector>

#include "../../include/imconv.h"

namespace {

struct Index {
    std::vector<int64_t> keys;
    std::vector<int32_t> slots;  // -1 = empty
    uint64_t mask;

    explicit Index(int64_t capacity) {
        uint64_t n = 16;
        while (n < static_cast<uint64_t>(capacity) * 2 + 2) n <<= 1;
        keys.assign(n, 0);
        slots.assign(n, -1);
        mask = n - 1;
    }
    static uint64_t hash(int64_t k) {
        uint64_t z = static_cast<uint64_t>(k) * 0x9E3779B97F4A7C15ull;
        return z ^ (z >> 29);
    }
    int64_t find(int64_t k) const {
        for (uint64_t i = hash(k) & mask;; i = (i + 1) & mask) {
            if (slots[i] < 0) return -1;
            if (keys[i] == k) return static_cast<int64_t>(i);
        }
    }
    void put(int64_t k, int32_t slot) {
        uint64_t i = hash(k) & mask;
        while (slots[i] >= 0) i = (i + 1) & mask;
        keys[i] = k;
        slots[i] = slot;
    }
    void erase_at(uint64_t i) {  // backward-shift deletion
        slots[i] = -1;
        for (uint64_t j = (i + 1) & mask; slots[j] >= 0; j = (j + 1) & mask) {
            const uint64_t h = hash(keys[j]) & mask;
            const bool move = (i <= j) ? (h <= i || h > j) : (h <= i && h > j);
            if (move) {
                keys[i] = keys[j];
                slots[i] = slots[j];
                slots[j] = -1;
                i = j;
            }
        }
    }
};

}  // namespace

extern "C" int imconv_lru_simulate(const int64_t *keys, int64_t count, int64_t capacity, int64_t *hits_out,
                                   int64_t *misses_out) {
    if (!hits_out || !misses_out || count < 0 || (count > 0 && !keys)) return IMCONV_EINVAL;
    if (capacity <= 0) {
        *hits_out = 0;
        *misses_out = count;
        return 0;
    }
    if (capacity > (1ll << 30)) return IMCONV_EINVAL;
    Index idx(capacity);
    std::vector<int64_t> slot_key(static_cast<size_t>(capacity));
    std::vector<int32_t> nxt(static_cast<size_t>(capacity) + 2), prv(static_cast<size_t>(capacity) + 2);
    const int32_t head = static_cast<int32_t>(capacity), tail = static_cast<int32_t>(capacity + 1);
    nxt[head] = tail;
    prv[tail] = head;
    int32_t filled = 0;
    int64_t hits = 0;
    for (int64_t t = 0; t < count; ++t) {
        const int64_t k = keys[t];
        int32_t slot;
        const int64_t pos = idx.find(k);
        if (pos >= 0) {
            ++hits;
            slot = idx.slots[static_cast<size_t>(pos)];
            nxt[prv[slot]] = nxt[slot];
            prv[nxt[slot]] = prv[slot];
        } else {
            if (filled < capacity) {
                slot = filled++;
            } else {
                slot = nxt[head];  // least recently used
                idx.erase_at(static_cast<uint64_t>(idx.find(slot_key[slot])));
                nxt[head] = nxt[slot];
                prv[nxt[slot]] = head;
            }
            slot_key[slot] = k;
            idx.put(k, slot);
        }
        prv[slot] = prv[tail];
        nxt[slot] = tail;
        nxt[prv[slot]] = slot;
        prv[tail] = slot;
    }
    *hits_out = hits;
    *misses_out = count - hits;
    return 0;
}
