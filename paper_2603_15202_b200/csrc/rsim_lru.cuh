// rsim_lru.cuh -- exact LRU eviction over "touch runs" (finite capacity only).
//
// The reference evicts, while occupancy > capacity, the unpinned entry that is
// smallest in (last_touch asc, depth desc, chain key asc) -- the effective
// order of its lazy heap (kvcache.py:142-168). Every touch of an entry here
// comes from one of three events, each of which touches a whole chain prefix
// with a single timestamp T:
//   enqueue  keys[1..h]  at arrival t         (engine.py:275, kvcache.py:109-119)
//   finish   chain[1..L] at step end          (engine.py:361, kvcache.py:81-104)
//   API      keys[1..n]  at now               (PrefixCache.insert_keys)
// so instead of one heap item per touched key we log one 48-byte *run*
// (T, chain, depth range 1..dhi) per event, in a per-instance ring kept sorted
// by T. An entry is live in the run whose T equals its current touch; older
// runs containing it are stale for it. Eviction walks runs from the oldest,
// one equal-T group at a time, and inside a group visits items in (depth
// desc, key asc) order -- exactly the reference order -- checking liveness
// (present, touch == T, depth == d) and pins in batches of 32 with one
// lookup round trip per batch. A group whose items are all gone is retired
// from the ring head. Groups of more than 32 runs (many chains finishing in
// one step at the same end time) fall back to the exact table scan.
#pragma once
#include "rsim_cache.cuh"

struct __align__(16) Run {
    i64 T;        // touch time of the event
    i64 a, oa;    // chain key offsets: prefix keys ckeys[a..a+B), output keys okeys[oa..]; kind 1: arena[a..]
    int B, dhi;   // prefix length, depth range 1..dhi
    int kind, pad;
};

__device__ __forceinline__ u64 run_key(const Params &P, const Run &r, int d) {   // d is 1-based
    if (r.kind == 1) return P.arena[r.a + d - 1];
    return d <= r.B ? P.ckeys[r.a + d - 1] : P.okeys[r.oa + d - 1 - r.B];
}

// Append one run, keeping the ring sorted by T (warp-collective; lane 0 writes).
// Updates the caller's Inst copy s (uniform across lanes).
__device__ void run_add(const Params &P, Inst &s, int gi, const Run &r, int lane, int &werr) {
    if (P.cap < 0 || P.runs == nullptr) return;
    Run *R = P.runs + ((size_t)gi << P.rlog2);
    const i64 mask = (1LL << P.rlog2) - 1;
    const i64 head = s.r_head, tail = s.r_tail;
    if (tail - head > mask) { werr = DEV_E_TABLE_FULL; return; }
    if (tail == head || r.T >= s.r_tailT) {
        if (lane == 0) R[tail & mask] = r;
        s.r_tail = tail + 1;
        s.r_tailT = r.T;
        __syncwarp();
        return;
    }
    // runs at the tail with a later T move up by one (few: the step in flight's finishes)
    i64 pos = tail;
    for (;;) {
        const i64 p = pos - 1 - lane;
        const bool gt = p >= head && R[p & mask].T > r.T;
        const u32 m = __ballot_sync(FULL, gt);
        const int c = m == FULL ? 32 : __ffs(~m) - 1;
        pos -= c;
        if (c < 32) break;
    }
    for (i64 q = tail - 1; q >= pos; q -= 32) {
        const i64 p = q - lane;
        Run v;
        if (p >= pos) v = R[p & mask];
        __syncwarp();
        if (p >= pos) R[(p + 1) & mask] = v;
        __syncwarp();
    }
    if (lane == 0) R[pos & mask] = r;
    s.r_tail = tail + 1;
    __syncwarp();
}

// Delete `key` (present) from the table: lookup + backward shift (lane 0).
__device__ __forceinline__ void delete_key(const Table &T, u64 key) {
    const int slot = tab_find(T, key);
    if (slot >= 0) tab_delete(T, (u32)slot);
}

// Evict down to capacity in exact reference order. Returns false when a group
// is too large for the run walk (the caller then uses the table scan).
__device__ bool evict_runs(const Params &P, const Table &T, Inst &s, int gi, i64 &occ, int lane, int &werr) {
    Run *R = P.runs + ((size_t)gi << P.rlog2);
    const i64 mask = (1LL << P.rlog2) - 1;
    i64 need = occ - P.cap;
    i64 pos = s.r_head;
    bool head_clean = true;
    __threadfence();                                   // order preceding RED touch/pin updates
    while (need > 0) {
        if (pos >= s.r_tail) { werr = DEV_E_CACHE_FULL; return true; }
        const i64 p = pos + lane;
        Run rr;
        rr.T = RSIM_NONE; rr.a = 0; rr.oa = 0; rr.B = 0; rr.dhi = 0; rr.kind = 0; rr.pad = 0;
        if (p < s.r_tail) rr = R[p & mask];
        const i64 T0 = __shfl_sync(FULL, rr.T, 0);
        const u32 gm = __ballot_sync(FULL, p < s.r_tail && rr.T == T0);
        if (gm == FULL) return false;                  // > 31 runs share T: fall back to the scan
        const int ng = __ffs(~gm) - 1;
        int maxd = __reduce_max_sync(FULL, lane < ng ? rr.dhi : 0);
        bool alive = false;                            // live items of the group left in place
        // K depth levels per batch, lanes = (run r, level l); order (depth desc, key asc)
        const int K = 32 / ng;
        int d0 = maxd;
        for (; d0 >= 1 && need > 0; d0 -= K) {
            const int r = lane % ng, l = lane / ng;
            const int d = d0 - l;
            const int dh = __shfl_sync(FULL, rr.dhi, r);
            Run rk;
            rk.T = T0;
            rk.a = __shfl_sync(FULL, rr.a, r); rk.oa = __shfl_sync(FULL, rr.oa, r);
            rk.B = __shfl_sync(FULL, rr.B, r); rk.kind = __shfl_sync(FULL, rr.kind, r);
            rk.dhi = dh; rk.pad = 0;
            const bool act = l < K && d >= 1 && d <= dh;
            const u64 key = act ? run_key(P, rk, d) : 0;
            // duplicates (shared prefixes of different chains) collapse to the lowest lane
            const u32 am = __ballot_sync(FULL, act);
            bool lead = false;
            if (act) { const u32 peers = __match_any_sync(am, key); lead = (__ffs(peers) - 1) == lane; }
            bool live = false, evictable = false;
            if (lead) {
                const int slot = tab_find(T, key);
                if (slot >= 0) {
                    const Meta m = load_meta(T.m + slot);
                    live = m.touch == T0 && m.depth == d;
                    evictable = live && m.pin <= 0;
                }
            }
            // rank in (depth desc, key asc) among the batch's evictable leaders: lanes are
            // level-major (depth desc); inside one level keys are compared directly
            const bool cand = evictable;
            const u32 cmask = __ballot_sync(FULL, cand);
            int rank = __popc(cmask & ((l * ng >= 32) ? FULL : ((1u << (l * ng)) - 1u)));
            if (ng > 1) {
#pragma unroll 1
                for (int o = 0; o < ng; o++) {
                    const int src = l * ng + o;
                    const u64 ok = __shfl_sync(FULL, key, src < 32 ? src : 31);
                    if (cand && src < 32 && src != lane && ((cmask >> src) & 1u) && ok < key) rank++;
                }
            }
            const i64 ncand = __popc(__ballot_sync(FULL, cand));
            const bool take = cand && rank < need;
            const i64 ntake = ncand < need ? ncand : need;
            alive = alive || __any_sync(FULL, live && !take);
            // delete the victims (order among them is irrelevant once chosen)
            u32 tm = __ballot_sync(FULL, take);
            while (tm) {
                const int l2 = __ffs(tm) - 1;
                tm &= tm - 1;
                const u64 vk = __shfl_sync(FULL, key, l2);
                if (lane == 0) delete_key(T, vk);
                __syncwarp();
            }
            occ -= ntake;
            need -= ntake;
        }
        if (d0 >= 1) alive = true;                     // levels below were not examined
        if (!alive && head_clean && pos == s.r_head) s.r_head = pos + ng;
        else head_clean = false;
        pos += ng;
    }
    return true;
}
