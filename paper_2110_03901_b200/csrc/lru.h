// lru.h -- fully-associative LRU over int64 keys (host C++), shared by the
// reference-compatible replay (imconv_lru_simulate, lru.cpp) and the B200
// DRAM-traffic predictor (imconv_predict_traffic, imconv_api.cu).
//
// Flat open-addressing index (key -> slot) plus an intrusive recency list:
// O(1) per access, no per-access allocation.  Each slot carries a dirty bit so
// a write-back cache (L2) can count the dirty lines it evicts.
#pragma once
#include <cstdint>
#include <vector>

namespace imconv {

struct LruIndex {
    std::vector<int64_t> keys;
    std::vector<int32_t> slots;  // -1 = empty
    uint64_t mask;

    explicit LruIndex(int64_t capacity) {
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

class LineLRU {
  public:
    explicit LineLRU(int64_t capacity)
        : cap_(capacity), idx_(capacity), key_(static_cast<size_t>(capacity)), dirty_(static_cast<size_t>(capacity)),
          nxt_(static_cast<size_t>(capacity) + 2), prv_(static_cast<size_t>(capacity) + 2) {
        head_ = static_cast<int32_t>(capacity);
        tail_ = static_cast<int32_t>(capacity + 1);
        nxt_[head_] = tail_;
        prv_[tail_] = head_;
    }
    // Touch `key`; `write` marks the line dirty.  Returns true on a hit.
    bool access(int64_t key, bool write) {
        int32_t slot;
        bool hit;
        const int64_t pos = idx_.find(key);
        if (pos >= 0) {
            hit = true;
            slot = idx_.slots[static_cast<size_t>(pos)];
            nxt_[prv_[slot]] = nxt_[slot];
            prv_[nxt_[slot]] = prv_[slot];
        } else {
            hit = false;
            if (filled_ < cap_) {
                slot = filled_++;
            } else {
                slot = nxt_[head_];  // least recently used
                if (dirty_[slot]) ++dirty_evictions_;
                idx_.erase_at(static_cast<uint64_t>(idx_.find(key_[slot])));
                nxt_[head_] = nxt_[slot];
                prv_[nxt_[slot]] = head_;
            }
            key_[slot] = key;
            dirty_[slot] = 0;
            idx_.put(key, slot);
        }
        if (write) dirty_[slot] = 1;
        prv_[slot] = prv_[tail_];
        nxt_[slot] = tail_;
        nxt_[prv_[slot]] = slot;
        prv_[tail_] = slot;
        return hit;
    }
    int64_t dirty_evictions() const { return dirty_evictions_; }
    int64_t dirty_resident() const {
        int64_t d = 0;
        for (int32_t i = 0; i < filled_; ++i) d += dirty_[i];
        return d;
    }

  private:
    int64_t cap_;
    LruIndex idx_;
    std::vector<int64_t> key_;
    std::vector<uint8_t> dirty_;
    std::vector<int32_t> nxt_, prv_;
    int32_t head_ = 0, tail_ = 0, filled_ = 0;
    int64_t dirty_evictions_ = 0;
};

}  // namespace imconv
