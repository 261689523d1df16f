// rsim_cache.cuh -- warp-cooperative KV$ prefix index (one open-addressing
// table per instance). Semantics follow PrefixCache (reference kvcache.py):
//   match      = longest present prefix               (kvcache.py:65-74)
//   insert     = create or touch=max(touch, now)      (kvcache.py:81-104)
//   touch/pin  = on keys[:upto]                       (kvcache.py:109-130)
//   unpin      = -1, error if not pinned              (kvcache.py:132-138)
//   evict      = while occupancy > capacity remove the smallest unpinned entry
//                in (touch asc, depth desc, key asc) order (kvcache.py:142-168;
//                that order is the reference lazy heap's effective total order)
// Only the owning warp touches an instance's table during a launch, so the
// only races are between lanes of one warp; duplicate keys inside a 32-key
// chunk are collapsed with __match_any_sync and slot claims are arbitrated
// the same way. Loads use ld.global.cg so a lane never reads a stale L1 line.
#pragma once
#include "rsim_device.cuh"

struct Table {
    u64 *k; Meta *m; u32 mask; int slog2; u64 empty;
};

__device__ __forceinline__ Table table_of(const Params &P, int gi) {
    Table t;
    t.k = P.tkeys + ((size_t)gi << P.slog2);
    t.m = P.tmeta + ((size_t)gi << P.slog2);
    t.mask = (1u << P.slog2) - 1u;
    t.slog2 = P.slog2;
    t.empty = P.empty;
    return t;
}

// Linear probing, four slots per round trip (the four loads are independent).
__device__ __forceinline__ int tab_find(const Table &T, u64 key) {
    u32 i = tab_home(key, T.slog2);
#pragma unroll 1
    for (;;) {
        u64 a0 = __ldcg(T.k + i);
        u64 a1 = __ldcg(T.k + ((i + 1) & T.mask));
        u64 a2 = __ldcg(T.k + ((i + 2) & T.mask));
        u64 a3 = __ldcg(T.k + ((i + 3) & T.mask));
        if (a0 == key) return (int)i;
        if (a0 == T.empty) return -1;
        if (a1 == key) return (int)((i + 1) & T.mask);
        if (a1 == T.empty) return -1;
        if (a2 == key) return (int)((i + 2) & T.mask);
        if (a2 == T.empty) return -1;
        if (a3 == key) return (int)((i + 3) & T.mask);
        if (a3 == T.empty) return -1;
        i = (i + 4) & T.mask;
    }
}

__device__ __forceinline__ Meta load_meta(const Meta *p) {
    Meta m;
    m.touch = __ldcg(&p->touch);
    m.depth = __ldcg(&p->depth);
    m.pin = __ldcg(&p->pin);
    return m;
}

// Longest present prefix of keys[0..B) (match_keys). Lane j probes depth j;
// the hit mask's leading ones are the match. Beyond 32 present blocks a
// 32-ary search over depth finds the boundary (presence is monotone in depth
// by prefix closure, kvcache.py:4-7), so a 2048-block prompt costs ~4 rounds.
__device__ int warp_probe(const Table &T, const u64 *keys, int B, int lane) {
    bool f = false;
    if (lane < B) f = tab_find(T, keys[lane]) >= 0;
    u32 m = __ballot_sync(FULL, f);
    if (m != FULL) return __ffs(~m) - 1;
    if (B <= 32) return 32;
    int lo = 32, hi = B;
    while (lo < hi) {
        int span = hi - lo, d;
        bool valid;
        if (span <= 32) { d = lo + lane; valid = lane < span; }
        else { d = lo + (int)(((i64)lane * span) >> 5); valid = true; }
        f = valid && tab_find(T, keys[d]) >= 0;
        m = __ballot_sync(FULL, f);
        u32 vm = __ballot_sync(FULL, valid);
        u32 miss = ~m & vm;
        int fm = miss ? __ffs(miss) - 1 : -1;
        if (fm == 0) break;                       // depth lo absent -> match = lo
        int last_ok = fm < 0 ? 31 - __clz(vm) : fm - 1;
        int d_ok = __shfl_sync(FULL, d, last_ok);
        int d_miss = __shfl_sync(FULL, d, fm < 0 ? 0 : fm);
        lo = d_ok + 1;
        if (fm > 0) hi = d_miss;
    }
    return lo;
}

// touch keys[:h] at now and pin them (InstanceSim.enqueue, engine.py:275-276).
__device__ void warp_touch_pin(const Table &T, const u64 *keys, int h, i64 now, int lane, int &werr) {
    for (int j0 = 0; j0 < h; j0 += 32) {
        int j = j0 + lane;
        bool act = j < h;
        u64 key = act ? keys[j] : 0;
        u32 am = __ballot_sync(FULL, act);
        if (act) {
            u32 peers = __match_any_sync(am, key);
            if (__ffs(peers) - 1 == lane) {
                int s = tab_find(T, key);
                if (s < 0) werr = DEV_E_INVARIANT;
                else {
                    Meta *mp = T.m + s;
                    i64 t0 = __ldcg(&mp->touch);
                    if (now > t0) mp->touch = now;
                    mp->pin = __ldcg(&mp->pin) + __popc(peers);
                }
            }
        }
        __syncwarp();
    }
    werr = __reduce_max_sync(FULL, werr);
}

// unpin keys[:h] (engine.py:360 -> kvcache.py:132-138)
__device__ void warp_unpin(const Table &T, const u64 *keys, int h, int lane, int &werr) {
    for (int j0 = 0; j0 < h; j0 += 32) {
        int j = j0 + lane;
        bool act = j < h;
        u64 key = act ? keys[j] : 0;
        u32 am = __ballot_sync(FULL, act);
        if (act) {
            u32 peers = __match_any_sync(am, key);
            if (__ffs(peers) - 1 == lane) {
                int s = tab_find(T, key);
                int cnt = __popc(peers);
                if (s < 0) werr = DEV_E_INVARIANT;
                else {
                    int p = __ldcg(&T.m[s].pin);
                    if (p < cnt) werr = DEV_E_INVARIANT;
                    else T.m[s].pin = p - cnt;
                }
            }
        }
        __syncwarp();
    }
    werr = __reduce_max_sync(FULL, werr);
}

// Insert (or touch) one chunk of <= 32 keys; lane j carries key/depth.
// Returns the number of newly created entries.
__device__ int warp_insert_chunk(const Table &T, bool act, u64 key, int depth, i64 now, int lane) {
    u32 am = __ballot_sync(FULL, act);
    bool lead = false;
    if (act) {
        u32 peers = __match_any_sync(am, key);
        lead = (__ffs(peers) - 1) == lane;   // first occurrence creates (its depth), kvcache.py:88-91
    }
    bool pend = lead, created = false;
    u32 pos = lead ? tab_home(key, T.slog2) : 0;
    int slot = -1;
    while (__ballot_sync(FULL, pend)) {
        if (pend) {
            for (;;) {
                u64 v = __ldcg(T.k + pos);
                if (v == key) { slot = (int)pos; pend = false; break; }
                if (v == T.empty) break;
                pos = (pos + 1) & T.mask;
            }
        }
        u32 cm = __ballot_sync(FULL, pend);
        if (pend) {
            u32 peers = __match_any_sync(cm, pos);
            if (__ffs(peers) - 1 == lane) {
                T.k[pos] = key;
                slot = (int)pos; created = true; pend = false;
            } else {
                pos = (pos + 1) & T.mask;
            }
        }
        __syncwarp();
    }
    if (slot >= 0) {
        Meta *mp = T.m + slot;
        if (created) { mp->touch = now; mp->depth = depth; mp->pin = 0; }
        else { i64 t0 = __ldcg(&mp->touch); if (now > t0) mp->touch = now; }
    }
    __syncwarp();
    return __popc(__ballot_sync(FULL, created));
}

// Backward-shift deletion (no tombstones, so probe chains never degrade).
__device__ void tab_delete(const Table &T, u32 i) {
    u32 j = i;
    for (;;) {
        j = (j + 1) & T.mask;
        u64 kj = __ldcg(T.k + j);
        if (kj == T.empty) break;
        u32 h = tab_home(kj, T.slog2);
        bool between = (i <= j) ? (h > i && h <= j) : (h > i || h <= j);
        if (!between) {
            T.k[i] = kj;
            T.m[i] = load_meta(T.m + j);
            i = j;
        }
    }
    T.k[i] = T.empty;
}

__device__ __forceinline__ bool lru_before(i64 t, int d, u64 k, i64 bt, int bd, u64 bk) {
    return t < bt || (t == bt && (d > bd || (d == bd && k < bk)));
}

// Exact LRU eviction down to capacity (kvcache.py:142-168): repeatedly
// remove the smallest unpinned entry in (touch asc, depth desc, key asc).
// Full-table warp scan per victim; the minimum is always a leaf, so prefix
// closure is preserved.
__device__ void warp_evict(const Table &T, i64 cap, i64 &occ, int lane, int &werr) {
    const u32 S = T.mask + 1;
    while (occ > cap) {
        i64 bt = RSIM_NONE; int bd = -1; u64 bk = ~0ULL; int bs = -1;
        for (u32 i = lane; i < S; i += 32) {
            u64 k = __ldcg(T.k + i);
            if (k == T.empty) continue;
            Meta m = load_meta(T.m + i);
            if (m.pin > 0) continue;
            if (bs < 0 || lru_before(m.touch, m.depth, k, bt, bd, bk)) { bt = m.touch; bd = m.depth; bk = k; bs = (int)i; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            i64 t2 = __shfl_xor_sync(FULL, bt, o);
            int d2 = __shfl_xor_sync(FULL, bd, o);
            u64 k2 = __shfl_xor_sync(FULL, bk, o);
            int s2 = __shfl_xor_sync(FULL, bs, o);
            if (s2 >= 0 && (bs < 0 || lru_before(t2, d2, k2, bt, bd, bk))) { bt = t2; bd = d2; bk = k2; bs = s2; }
        }
        if (bs < 0) { werr = DEV_E_CACHE_FULL; return; }
        if (lane == 0) tab_delete(T, (u32)bs);
        __syncwarp();
        occ--;
    }
}
