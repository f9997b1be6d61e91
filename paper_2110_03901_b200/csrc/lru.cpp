// lru.cpp -- host-side LRU replay behind blocksched.reuse_traffic.
//
// The reference evaluates its subtile orders with a fully-associative LRU
// over gathered element keys (_native.pyx:102-149, blocksched.py:131-151).
// That is an inherently sequential analysis model, not device work, so it
// stays on the host in C++ (lru.h: O(1) per access, no per-access allocation).
#include <cstdint>
#include <vector>

#include "../../include/imconv.h"
#include "lru.h"

extern "C" int imconv_lru_simulate(const int64_t *keys, int64_t count, int64_t capacity, int64_t *hits_out,
                                   int64_t *misses_out) {
    if (!hits_out || !misses_out || count < 0 || (count > 0 && !keys)) return IMCONV_EINVAL;
    if (capacity <= 0) {
        *hits_out = 0;
        *misses_out = count;
        return 0;
    }
    if (capacity > (1ll << 30)) return IMCONV_EINVAL;
    imconv::LineLRU lru(capacity);
    int64_t hits = 0;
    for (int64_t t = 0; t < count; ++t) hits += lru.access(keys[t], false) ? 1 : 0;
    *hits_out = hits;
    *misses_out = count - hits;
    return 0;
}
