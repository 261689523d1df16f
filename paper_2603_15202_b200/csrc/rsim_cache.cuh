// rsim_cache.cuh -- warp-cooperative KV$ prefix index (one open-addressing
// table per instance). Semantics follow PrefixCache (reference kvcache.py):
//   match      = longest present prefix               (kvcache.py:65-74)
//   insert     = create or touch=max(touch, now)      (kvcache.py:81-104)
//   touch/pin  = on keys[:upto]                       (kvcache.py:109-130)
//   unpin      = -1 on keys[:upto]                    (kvcache.py:132-138)
//   evict      = while occupancy > capacity remove the smallest unpinned entry
//                in (touch asc, depth desc, key asc) order (kvcache.py:142-168;
//                that order is the reference lazy heap's effective total order)
//
// Latency is the budget here (one decision is a serial chain of these calls),
// so every operation is shaped to cost one memory round trip per 128 keys:
//  * a warp handles 128 chain depths per round, 4 per lane, all loads in flight;
//  * linear probing reads an aligned 16-byte slot pair per load (tables run at
//    <= 3/4 load, usually far below, so the home pair nearly always decides);
//  * an instance's table is written only by its owning warp (one SM) during a
//    launch, so slot claims are plain stores arbitrated among the warp's own
//    lanes (__match_any_sync); key probes read L2 directly (ld.global.cg);
//  * touch / pin / unpin are fire-and-forget atomics (RED) on the metadata:
//    max and +/- are commutative, so no read-modify-write round trip is
//    needed; metadata is only ever read through L2 (ld.global.cg).
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

__device__ __forceinline__ ulonglong2 ld_pair(const Table &T, u32 i) {
    // L2 only (ld.global.cg): table lines have little reuse inside one SM, and not allocating
    // them keeps L1 for the engine's queue / running records (measured: -7 % per decision, chat1024)
    return __ldcg(reinterpret_cast<const ulonglong2 *>(T.k) + (i >> 1));
}
// L1-allocating pair load for the insert / touch paths, which re-read the lines they just
// looked up (claims). Safe: an instance's table is written only by its owning warp's SM.
__device__ __forceinline__ ulonglong2 ld_pair_l1(const Table &T, u32 i) {
    return __ldca(reinterpret_cast<const ulonglong2 *>(T.k) + (i >> 1));
}

// Evaluate one aligned pair starting the probe at slot i.
// st: 0 found (returns slot), 1 absent (returns the first EMPTY slot), 2 continue (returns next i)
__device__ __forceinline__ u32 eval_pair(const Table &T, ulonglong2 pr, u32 i, u64 key, int &st) {
    if ((i & 1u) == 0) {
        if (pr.x == key) { st = 0; return i; }
        if (pr.x == T.empty) { st = 1; return i; }
    }
    const u32 j = i | 1u;
    if (pr.y == key) { st = 0; return j; }
    if (pr.y == T.empty) { st = 1; return j; }
    st = 2;
    return (j + 1) & T.mask;
}

// Finish a probe that did not resolve in its first pair. Out of line and with
// scalar arguments only (no caller object has its address taken, so callers
// keep the table and the status in registers); returns (status << 32) | slot.
__device__ __noinline__ u64 probe_rest_v(u64 *tk, u32 mask, u64 empty, u32 i, u64 key) {
    Table T;
    T.k = tk; T.m = nullptr; T.mask = mask; T.slog2 = 0; T.empty = empty;
    for (;;) {
        int st;
        ulonglong2 pr = ld_pair(T, i);
        u32 r = eval_pair(T, pr, i, key, st);
        if (st != 2) return ((u64)(u32)st << 32) | r;
        i = r;
    }
}
__device__ __forceinline__ u32 probe_rest(const Table &T, u32 i, u64 key, int &st) {
    const u64 v = probe_rest_v(T.k, T.mask, T.empty, i, key);
    st = (int)(v >> 32);
    return (u32)v;
}

__device__ __forceinline__ int tab_find(const Table &T, u64 key) {
    int st;
    u32 i = tab_home(key, T.slog2);
    u32 r = eval_pair(T, ld_pair_l1(T, i), i, key, st);
    if (st == 2) r = probe_rest(T, r, key, st);
    return st == 0 ? (int)r : -1;
}

__device__ __forceinline__ Meta load_meta(const Meta *p) {
    Meta m;
    m.touch = __ldcg(&p->touch);
    m.depth = __ldcg(&p->depth);
    m.pin = __ldcg(&p->pin);
    return m;
}

// Batched lookup of up to 128 keys (lane-major: key k of lane = depth 32k+lane).
// slot[k] = found slot or -1; freepos[k] = first EMPTY slot when absent.
__device__ __forceinline__ void find128(const Table &T, const u64 kk[4], const bool act[4], int slot[4],
                                        u32 freepos[4]) {
    ulonglong2 pr[4];
    u32 home[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
        home[k] = tab_home(kk[k], T.slog2);
        pr[k] = act[k] ? ld_pair_l1(T, home[k]) : make_ulonglong2(0ULL, 0ULL);   // unconditional: stays in registers
    }
#pragma unroll
    for (int k = 0; k < 4; k++) {
        slot[k] = -1;
        freepos[k] = 0;
        if (act[k]) {
            int st;
            u32 r = eval_pair(T, pr[k], home[k], kk[k], st);
            if (st == 2) r = probe_rest(T, r, kk[k], st);
            if (st == 0) slot[k] = (int)r; else freepos[k] = r;
        }
    }
}

// Hit masks for the first 128 depths of NI instances at once (loads of all
// instances in flight together). m[s][k] bit lane = depth 32k+lane present.
// Branch-free evaluation of a key's first aligned pair (linear probing from
// slot i): f = found in the pair, c = pair full of other keys (probe goes on).
__device__ __forceinline__ void eval_first(const Table &T, ulonglong2 pr, u32 i, u64 key, bool &f, bool &c) {
    const bool ev = (i & 1u) == 0;
    const bool xk = ev && pr.x == key, xe = ev && pr.x == T.empty;
    f = xk || (!xe && pr.y == key);
    c = !xk && !xe && pr.y != key && pr.y != T.empty;
}

template <int NI>
__device__ __forceinline__ void probe128(const Table *T, const u64 kk[4], const u32 hm[4], int B, int lane,
                                         u32 m[NI][4], int slot[NI][4]) {
    ulonglong2 pr[NI][4];
    const int nk = (B + 31) >> 5;                       // warp-uniform: depth slots in use
#pragma unroll
    for (int s = 0; s < NI; s++)
#pragma unroll
        for (int k = 0; k < 4; k++)
            pr[s][k] = (k < nk && 32 * k + lane < B) ? ld_pair(T[s], hm[k]) : make_ulonglong2(0ULL, 0ULL);
#pragma unroll
    for (int s = 0; s < NI; s++)
#pragma unroll
        for (int k = 0; k < 4; k++) {
            slot[s][k] = -1;
            m[s][k] = 0;
            if (k < nk) {
                bool f = false, c = false;
                if (32 * k + lane < B) eval_first(T[s], pr[s][k], hm[k], kk[k], f, c);
                if (__any_sync(FULL, c) && c) {     // rare: the home pair is full of other keys
                    int st;
                    const u32 r = probe_rest(T[s], (hm[k] | 1u) + 1u & T[s].mask, kk[k], st);
                    f = st == 0;
                    if (f) slot[s][k] = (int)r;
                } else if (f) {
                    slot[s][k] = (int)((hm[k] & 1u) == 0 && pr[s][k].x == kk[k] ? hm[k] : hm[k] | 1u);
                }
                m[s][k] = __ballot_sync(FULL, f);
            }
        }
}

__device__ __forceinline__ int lead_hits(const u32 m[4]) {   // leading present depths
    if (m[0] != FULL) return __ffs(~m[0]) - 1;
    if (m[1] != FULL) return 32 + __ffs(~m[1]) - 1;
    if (m[2] != FULL) return 64 + __ffs(~m[2]) - 1;
    if (m[3] != FULL) return 96 + __ffs(~m[3]) - 1;
    return 128;
}

// Longest present prefix beyond the first 128 depths: 128-ary search over
// depth (presence is monotone in depth by prefix closure, kvcache.py:4-7),
// ~3 rounds for a 2048-block prompt. keys = the request's chain keys.
__device__ __noinline__ int deep_match_v(u64 *tk, u32 mask, int slog2, u64 empty, const u64 *keys, int B, int lane) {
    Table T;
    T.k = tk; T.m = nullptr; T.mask = mask; T.slog2 = slog2; T.empty = empty;
    int lo = 128, hi = B;
    while (lo < hi) {
        const int span = hi - lo;
        int d[4];
        bool valid[4], f[4];
        u64 kk[4];
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int idx = 32 * k + lane;
            if (span <= 128) { d[k] = lo + idx; valid[k] = idx < span; }
            else { d[k] = lo + (int)(((i64)idx * span) >> 7); valid[k] = true; }
            kk[k] = valid[k] ? keys[d[k]] : 0;
        }
        int slot[4];
        u32 fp[4];
        find128(T, kk, valid, slot, fp);
        u32 miss[4], vm[4];
#pragma unroll
        for (int k = 0; k < 4; k++) {
            f[k] = valid[k] && slot[k] >= 0;
            miss[k] = __ballot_sync(FULL, valid[k] && !f[k]);
            vm[k] = __ballot_sync(FULL, valid[k]);
        }
        int fm = -1, last = -1;
#pragma unroll
        for (int k = 3; k >= 0; k--) if (vm[k] && last < 0) last = 32 * k + 31 - __clz(vm[k]);
#pragma unroll
        for (int k = 0; k < 4; k++) if (miss[k] && fm < 0) fm = 32 * k + __ffs(miss[k]) - 1;
        if (fm == 0) break;                                   // depth lo absent: match = lo
        const int ok = fm < 0 ? last : fm - 1;
        const int d_ok = __shfl_sync(FULL, d[ok >> 5], ok & 31);
        if (fm > 0) hi = __shfl_sync(FULL, d[fm >> 5], fm & 31);
        lo = d_ok + 1;
    }
    return lo;
}
__device__ __forceinline__ int deep_match(const Table &T, const u64 *keys, int B, int lane) {
    return deep_match_v(T.k, T.mask, T.slog2, T.empty, keys, B, lane);
}

// Longest present prefix of one instance (match_keys) -- the API / batch path.
__device__ int warp_probe(const Table &T, const u64 *keys, int B, int lane) {
    u64 kk[4];
#pragma unroll
    for (int k = 0; k < 4; k++) kk[k] = (32 * k + lane < B) ? keys[32 * k + lane] : 0;
    u32 m[1][4], hm[4];
    int sl[1][4];
#pragma unroll
    for (int k = 0; k < 4; k++) hm[k] = tab_home(kk[k], T.slog2);
    probe128<1>(&T, kk, hm, B, lane, m, sl);
    int h = lead_hits(m[0]);
    if (h < 128) return min(h, B);
    if (B <= 128) return B;
    return deep_match(T, keys, B, lane);
}

// touch keys[:h] at now and pin them (InstanceSim.enqueue, engine.py:275-276).
// kk0 holds the first 128 keys (already in registers from the probe); slot0,
// when non-null, holds their slots as found by that probe (no lookup needed).
__device__ void warp_touch_pin(const Table &T, const u64 *keys, const u64 kk0[4], const int *slot0, int h, i64 now,
                               int lane, int &werr) {
    for (int j0 = 0; j0 < h; j0 += 128) {
        u64 kk[4];
        bool act[4];
        int slot[4];
        u32 fp[4];
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int j = j0 + 32 * k + lane;
            act[k] = j < h;
            kk[k] = j0 == 0 ? kk0[k] : (act[k] ? keys[j] : 0);
        }
        if (j0 == 0 && slot0 != nullptr) {
#pragma unroll
            for (int k = 0; k < 4; k++) slot[k] = slot0[k];
        } else {
            find128(T, kk, act, slot, fp);
        }
#pragma unroll
        for (int k = 0; k < 4; k++) {
            if (!act[k]) continue;
            if (slot[k] < 0) { werr = DEV_E_INVARIANT; continue; }
            Meta *mp = T.m + slot[k];
            atomicMax(&mp->touch, now);
            atomicAdd(&mp->pin, 1);
        }
    }
    werr = __reduce_max_sync(FULL, werr);
}

// Claim slots for the absent keys of a 128-key batch with plain stores. One
// k-slot at a time, every claimant re-probes from its key's home (L1), so a
// duplicate key already inserted or a slot taken by an earlier claim is seen;
// lanes aiming at the same EMPTY slot are arbitrated with __match_any_sync.
__device__ __forceinline__ void claim128(const Table &T, const u64 kk[4], const bool need[4], int slot[4],
                                         bool created[4], int lane) {
#pragma unroll
    for (int k = 0; k < 4; k++) {
        bool pend = need[k];
        while (__ballot_sync(FULL, pend)) {
            u32 pos = 0;
            if (pend) {
                int st;
                const u32 i = tab_home(kk[k], T.slog2);
                u32 r = eval_pair(T, ld_pair_l1(T, i), i, kk[k], st);
                if (st == 2) r = probe_rest(T, r, kk[k], st);
                if (st == 0) { slot[k] = (int)r; pend = false; }
                else pos = r;
            }
            const u32 cm = __ballot_sync(FULL, pend);
            if (pend) {
                const u32 peers = __match_any_sync(cm, pos);
                if (__ffs(peers) - 1 == lane) { T.k[pos] = kk[k]; slot[k] = (int)pos; created[k] = true; pend = false; }
            }
            __syncwarp();
        }
    }
}

// Fused _finish cache work (engine.py:357-361): unpin keys[:hb], then insert
// the full chain (prefix keys pk[0..B) then output keys ok[0..L-B)) at `now`.
// Returns the number of created entries.
__device__ int warp_unpin_insert(const Table &T, const u64 *pk, int B, const u64 *ok, int L, int hb, i64 now,
                                 int lane, int &werr) {
    int created_total = 0;
    for (int j0 = 0; j0 < L; j0 += 128) {
        u64 kk[4];
        bool act[4];
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int j = j0 + 32 * k + lane;
            act[k] = j < L;
            kk[k] = act[k] ? (j < B ? pk[j] : ok[j - B]) : 0;
        }
        int slot[4];
        u32 fp[4];
        find128(T, kk, act, slot, fp);
        bool created[4], need[4];
#pragma unroll
        for (int k = 0; k < 4; k++) { created[k] = false; need[k] = act[k] && slot[k] < 0; }
        claim128(T, kk, need, slot, created, lane);
#pragma unroll
        for (int k = 0; k < 4; k++) {
            if (!act[k]) continue;
            const int j = j0 + 32 * k + lane;
            Meta *mp = T.m + slot[k];
            if (created[k]) {
                Meta m; m.touch = now; m.depth = j + 1; m.pin = 0;
                *mp = m;
                if (j < hb) werr = DEV_E_INVARIANT;         // a pinned chain cannot be absent
            } else {
                atomicMax(&mp->touch, now);
                if (j < hb) atomicSub(&mp->pin, 1);
            }
            created_total += created[k];
        }
    }
    werr = __reduce_max_sync(FULL, werr);
    return __reduce_add_sync(FULL, created_total);
}

// Finish cache work of several requests of one engine step at once (legal
// when no eviction can occur in between: inserts, touches and unpins commute).
// Flattened over all chains, 128 keys per round: one load, one lookup and one
// claim round trip per round instead of per request.
struct FinBuf {
    i64 a[32], oa[32];
    u64 kx[32];                 // Ent.kx of each finisher
    int B[32], L[32], hb[32], pre[33];
    // a batch whose cache work was deferred past the current decision's publish
    // (rsim_engine.cuh: finish_or_defer): dnf finishers of local instance dsp / gi dgi, stamped dend
    int dnf, dgi, dsi, npark;   // ..., local index of that instance, batches parked (diagnostics)
    i64 dend;
    struct Inst *dsp;
    // the last commit's touch + pin of the hit chain (engine.py:275-276), run off the critical
    // path: before any finisher cache work of that instance and before the next commit
    int tpn, tpgi, tph, tpver;  // pending?, instance, hit blocks, instance tabver at commit
    i64 tpa, tpt;               // request chain key offset, touch time
    const u64 *tpkeys;          // the request's first 128 chain keys (its staging slot)
    const int *tpsl;            // their probe-found slots, or null
    struct Inst *tpsp;
    i64 lnext, lend;            // this warp's reserved step-log records [lnext, lend) (log_step)
};

__device__ int warp_finish_many(const Table &T, const u64 *ckeys, const u64 *okeys, const FinBuf &F, int nf, i64 now,
                                int lane, int &werr) {
    const int K = F.pre[nf];
    int created_total = 0;
    for (int x0 = 0; x0 < K; x0 += 128) {
        u64 kk[4];
        bool act[4];
        int dep[4];
        bool unp[4];
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int x = x0 + 32 * k + lane;
            act[k] = x < K;
            int f = 0;
            if (act[k])
                while (f + 1 < nf && F.pre[f + 1] <= x) f++;
            const int j = x - F.pre[f];
            // unconditional assignments (a conditionally assigned array goes to local memory)
            kk[k] = act[k] ? (j < F.B[f] ? ckeys[F.a[f] + j] : okeys[F.oa[f] + j - F.B[f]]) : 0ULL;
            dep[k] = act[k] ? j + 1 : 0;
            unp[k] = act[k] && j < F.hb[f];
        }
        int slot[4];
        u32 fp[4];
        find128(T, kk, act, slot, fp);
        bool created[4], need[4];
#pragma unroll
        for (int k = 0; k < 4; k++) { created[k] = false; need[k] = act[k] && slot[k] < 0; }
        claim128(T, kk, need, slot, created, lane);
#pragma unroll
        for (int k = 0; k < 4; k++) {
            if (!act[k]) continue;
            Meta *mp = T.m + slot[k];
            if (created[k]) {
                Meta m; m.touch = now; m.depth = dep[k]; m.pin = 0;
                *mp = m;
                if (unp[k]) werr = DEV_E_INVARIANT;
            } else {
                atomicMax(&mp->touch, now);
                if (unp[k]) atomicSub(&mp->pin, 1);
            }
            created_total += created[k];
        }
    }
    werr = __reduce_max_sync(FULL, werr);
    return __reduce_add_sync(FULL, created_total);
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

// Delete up to 32 present entries at once (lane l deletes key kv at slot v when del): the
// same key set as backward-shift deleting them one by one and again a table with no hole on
// any probe path, in a few round trips instead of ~4 dependent ones per key. Victims are
// first marked (a transient TOMB key); then every maximal run of slots from a victim to the
// next EMPTY is rebuilt by one lane: its live entries are re-inserted in slot order, each
// into the first free slot at or after its home (homes before the run count as its start),
// which never moves an entry forward; the rest of the run becomes EMPTY. Runs of different
// lanes are disjoint (each ends at an EMPTY slot); a victim inside another victim's run is
// left to that run's lane. A run longer than 64 slots (a bitmap) sends the whole batch to
// the one-at-a-time path. Only the owning warp touches the table: plain stores suffice.
#define RSIM_TOMB (~0ULL)
__device__ __forceinline__ void tab_place(u64 *tk, Meta *tm, u32 mask, int slog2, u32 v, u32 off, u64 k, u64 &occ) {
    if (k == RSIM_TOMB) return;
    const u32 u = (tab_home(k, slog2) - v) & mask;      // home offset; > off: home before v
    const u32 st = u <= off ? u : 0;
    const u32 t = (u32)(__ffsll((long long)(~occ & (~0ULL << st))) - 1);   // <= off
    occ |= 1ULL << t;
    if (t != off) {
        const u32 x = (v + off) & mask, y = (v + t) & mask;
        const ulonglong2 m = __ldcg(reinterpret_cast<const ulonglong2 *>(tm + x));
        tk[y] = k;
        *reinterpret_cast<ulonglong2 *>(tm + y) = m;
    }
}

__device__ __forceinline__ void tab_delete32(u64 *tk, Meta *tm, u32 mask, int slog2, u32 v, u64 kv, bool del, int lane) {
    if (!__any_sync(FULL, del)) return;
    if (del) tk[v] = RSIM_TOMB;
    __syncwarp();
    // the run [v, v + len): len = distance to the first EMPTY after v (8 slots per round trip;
    // the first window stays in registers for the rebuild)
    u32 len = 0;
    u64 w[8];
#pragma unroll
    for (int i = 0; i < 8; i++) w[i] = del ? __ldcg(tk + ((v + 1 + i) & mask)) : 0ULL;
    if (del) {
#pragma unroll
        for (int i = 7; i >= 0; i--) if (w[i] == 0ULL) len = 1 + (u32)i;
        for (u32 base = 9; len == 0 && base <= 64; base += 8) {
            u64 x[8];
#pragma unroll
            for (int i = 0; i < 8; i++) x[i] = __ldcg(tk + ((v + base + i) & mask));
#pragma unroll
            for (int i = 7; i >= 0; i--) if (x[i] == 0ULL) len = base + (u32)i;
        }
    }
    if (__any_sync(FULL, del && (len == 0 || len > 64))) {     // a long run: one key at a time
        if (del) tk[v] = kv;
        __syncwarp();
        Table T;
        T.k = tk; T.m = tm; T.mask = mask; T.slog2 = slog2; T.empty = 0ULL;
        for (u32 b = __ballot_sync(FULL, del); b; b &= b - 1) {
            const u64 key = __shfl_sync(FULL, kv, __ffs(b) - 1);
            if (lane == 0) {
                const int slot = tab_find(T, key);
                if (slot >= 0) tab_delete(T, (u32)slot);
            }
            __syncwarp();
        }
        return;
    }
    // a victim inside another victim's run belongs to that run
    bool lead = del;
    for (u32 b = __ballot_sync(FULL, del); b; b &= b - 1) {     // warp-uniform loop over the victims
        const int o = __ffs(b) - 1;
        const u32 vo = __shfl_sync(FULL, v, o), lo = __shfl_sync(FULL, len, o);
        const u32 dist = (v - vo) & mask;
        if (o != lane && dist != 0 && dist < lo) lead = false;
    }
    if (lead) {
        u64 occ = 0;                                    // offsets of the run already re-filled
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const u32 off = (u32)i + 1;
            if (off < len) tab_place(tk, tm, mask, slog2, v, off, w[i], occ);
        }
        for (u32 off = 9; off < len; off++) tab_place(tk, tm, mask, slog2, v, off, __ldcg(tk + ((v + off) & mask)), occ);
        for (u32 g = 0; g < len; g++)
            if (!((occ >> g) & 1ULL)) tk[(v + g) & mask] = 0ULL;
    }
    __syncwarp();
}

__device__ __forceinline__ bool lru_before(i64 t, int d, u64 k, i64 bt, int bd, u64 bk) {
    return t < bt || (t == bt && (d > bd || (d == bd && k < bk)));
}

// Exact LRU eviction down to capacity (kvcache.py:142-168): repeatedly
// remove the smallest unpinned entry in (touch asc, depth desc, key asc).
// Full-table warp scan per victim; the minimum is always a leaf, so prefix
// closure is preserved. A pinned-out table raises CacheFullError.
__device__ void warp_evict(const Table &T, i64 cap, i64 &occ, int lane, int &werr) {
    const u32 S = T.mask + 1;
    __threadfence();                     // order the preceding RED touch/pin updates
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
