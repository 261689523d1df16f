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
    if (tail - head > mask) { werr = DEV_E_RUNS_FULL; return; }
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

// Evict from the single run r (the oldest touch group, no other run shares its T), deepest
// depth first: the reference's (touch asc, depth desc, key asc) order restricted to one
// chain. Every event touches or pins a whole chain PREFIX (kvcache.py:81-138), so along the
// chain touch and pin never increase with depth (prefix closure, kvcache.py:4-7, keeps the
// present items a prefix too). Walking up from the deepest depth the items are therefore:
// absent or re-touched older than T (skipped: not live in this run), then live (touch == T)
// and unpinned -- the victims, in order --, then a first item that is pinned or newer, above
// which nothing in this run is evictable. 128 depths per round trip (plus one for the
// metadata); the victims go in batches of 32 (tab_delete32). Returns the run's new depth
// bound: everything deeper is known dead for this run.
__device__ __forceinline__ int evict_chain_body(const Params &P, const Table &T, const Run &r, i64 &need, int lane,
                                                bool &alive) {
    int d0 = r.dhi;
    while (d0 >= 1 && need > 0) {
        u64 kk[4];
        bool act[4];
        int slot[4];
        u32 fp[4];
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int d = d0 - (32 * k + lane);
            act[k] = d >= 1;
            kk[k] = act[k] ? run_key(P, r, d) : 0ULL;
        }
        find128(T, kk, act, slot, fp);
        // 0 skip, 1 victim, 2 newer (stop), 3 live but pinned (stop; the run stays)
        int cls[4];
#pragma unroll
        for (int k = 0; k < 4; k++) {
            cls[k] = 0;
            if (slot[k] >= 0) {
                const Meta m = load_meta(T.m + slot[k]);
                const int d = d0 - (32 * k + lane);
                if (m.touch > r.T) cls[k] = 2;
                else if (m.touch == r.T && m.depth == d) cls[k] = m.pin > 0 ? 3 : 1;
            }
        }
        // first stop in depth order (k major, lane minor), and the victims before it
        int stop = 128;
#pragma unroll
        for (int k = 3; k >= 0; k--) {
            const u32 sm = __ballot_sync(FULL, cls[k] >= 2);
            if (sm) stop = 32 * k + __ffs(sm) - 1;
        }
        const int ncand = __reduce_add_sync(FULL, (cls[0] == 1 && lane < stop) + (cls[1] == 1 && 32 + lane < stop) +
                                                      (cls[2] == 1 && 64 + lane < stop) + (cls[3] == 1 && 96 + lane < stop));
        const i64 ntake = ncand < need ? ncand : need;
        int taken = 0, last = -1;                      // victims taken so far in depth order; index of the last
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int idx = 32 * k + lane;
            const bool cand = cls[k] == 1 && idx < stop;
            const u32 cm = __ballot_sync(FULL, cand);
            const bool take = cand && taken + __popc(cm & lanemask_lt()) < ntake;
            const u32 tm = __ballot_sync(FULL, take);
            if (tm) last = 32 * k + 31 - __clz(tm);
            taken += __popc(tm);
#ifdef RSIM_STEP_PROFILE
            const long long cd = clock64();
            if (P.ctr != nullptr && lane == 0 && tm) { atomicAdd(P.ctr + 44, (u64)1); atomicAdd(P.ctr + 45, (u64)__popc(tm)); }
#endif
            // an earlier deletion of this batch may have shifted the slot (backward shifts)
            int sl = slot[k];
            if (taken > __popc(tm) && take) sl = tab_find(T, kk[k]);
            tab_delete32(T.k, T.m, T.mask, T.slog2, (u32)sl, kk[k], take, lane);
#ifdef RSIM_STEP_PROFILE
            if (P.ctr != nullptr && lane == 0 && tm) atomicAdd(P.ctr + 46, (u64)(clock64() - cd));
#endif
        }
        need -= ntake;
        if (ntake < ncand) {                           // capacity reached: victims remain live
            alive = true;
            return d0 - last - 1;
        }
        if (stop < 128) {                              // nothing above is evictable in this run
            int cs = cls[0];
#pragma unroll
            for (int k = 1; k < 4; k++) if ((stop >> 5) == k) cs = cls[k];
            alive = __shfl_sync(FULL, cs, stop & 31) == 3;
            return d0 - stop;
        }
        if (need == 0) {                               // done; what lies above is unknown
            alive = true;
            return d0 > 128 ? d0 - 128 : 0;
        }
        d0 -= 128;
    }
    return 0;
}

// Out of line with scalar arguments only (no caller object has its address taken); returns
// (victims << 32) | (alive << 31) | new depth bound.
__device__ __forceinline__ u64 evict_chain_v(const Params &P, u64 *tk, Meta *tmeta, u32 tmask, int slog2, i64 rT, i64 ra,
                                          i64 roa, int rB, int rkind, int rdhi, i64 need0, int lane) {
    Table T;
    T.k = tk; T.m = tmeta; T.mask = tmask; T.slog2 = slog2; T.empty = 0;
    Run r;
    r.T = rT; r.a = ra; r.oa = roa; r.B = rB; r.kind = rkind; r.dhi = rdhi; r.pad = 0;
    i64 need = need0;
    bool alive = false;
    const int nd = evict_chain_body(P, T, r, need, lane, alive);
    return ((u64)(need0 - need) << 32) | ((u64)alive << 31) | (u64)(u32)nd;
}

// Evict down to capacity in exact reference order. Returns false when a group
// is too large for the run walk (the caller then uses the table scan).
__device__ bool evict_runs(const Params &P, const Table &T, Inst &s, int gi, i64 &occ, int lane,
                                                int &werr) {
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
#ifdef RSIM_STEP_PROFILE
        if (P.ctr != nullptr && lane == 0) atomicAdd(P.ctr + 47, (u64)1);
#endif
        const int ng = __ffs(~gm) - 1;
        if (ng == 1) {                                 // one run: its live items are one depth range
            bool alive = false;
            const int dhi = __shfl_sync(FULL, rr.dhi, 0);
            const u64 res = evict_chain_v(P, T.k, T.m, T.mask, T.slog2, T0, __shfl_sync(FULL, rr.a, 0),
                                          __shfl_sync(FULL, rr.oa, 0), __shfl_sync(FULL, rr.B, 0),
                                          __shfl_sync(FULL, rr.kind, 0), dhi, need, lane);
            const int ndhi = (int)(res & 0x7fffffffu);
            alive = (res >> 31) & 1u;
            need -= (i64)(res >> 32);
            occ -= (i64)(res >> 32);
            if (lane == 0 && ndhi != dhi) R[pos & mask].dhi = ndhi;
            if (!alive && head_clean && pos == s.r_head) s.r_head = pos + 1;
            else head_clean = false;
            pos += 1;
            continue;
        }
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
            int slot = -1;
            if (lead) {
                slot = tab_find(T, key);
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
#ifdef RSIM_STEP_PROFILE
            const long long cd = clock64();
            if (P.ctr != nullptr && lane == 0) { atomicAdd(P.ctr + 44, (u64)1); atomicAdd(P.ctr + 45, (u64)ntake); }
#endif
            tab_delete32(T.k, T.m, T.mask, T.slog2, (u32)slot, key, take, lane);
#ifdef RSIM_STEP_PROFILE
            if (P.ctr != nullptr && lane == 0) atomicAdd(P.ctr + 46, (u64)(clock64() - cd));
#endif
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
