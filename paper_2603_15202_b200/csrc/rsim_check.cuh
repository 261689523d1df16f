// rsim_check.cuh -- ClusterConfig.debug_checks on the device.
//
// The reference runs, after every engine step when debug_checks is set
// (cluster.py:168-170):
//   InstanceSim.reconcile        (engine.py:248-258): the live aggregates
//       (running, queued, pending, total, dc) equal a recount over the slots;
//   PrefixCache.check_invariants (kvcache.py:178-194): occupancy <= capacity;
//       every entry has depth >= 1 and pin >= 0; every entry of depth > 1 has
//       its parent present at depth - 1, touched no earlier and pinned at least
//       as often (prefix closure, LRU-eviction safety, pins cover the path).
// With debug_checks the host replays one decision per launch and runs this
// kernel after each one (and after the drain), so a violation surfaces at the
// decision whose steps caused it, as RSIM_E_INVARIANT (InvariantError).
//
// The table stores no parent pointers (Meta is 16 B on the hot path), so the
// parent relation is recovered from the chains that put keys into an instance:
// the full chains (prefix + output keys, engine.py:363-372) of the requests
// routed to it, and the chains inserted through the PrefixCache API (segments
// of the key arena). A present key that no such chain names is reported too.
#pragma once
#include "rsim_cache.cuh"

// info codes (rsim_status message): what failed
enum {
    CHK_AGG = 1,          // reconcile: aggregates != recount
    CHK_ENTRY = 2,        // depth < 1 or pin < 0
    CHK_OCC = 3,          // occupancy counter != present entries
    CHK_CAP = 4,          // occupancy over capacity
    CHK_DEPTH = 5,        // key at chain position j does not have depth j + 1
    CHK_CLOSURE = 6,      // parent missing (prefix closure violated)
    CHK_TOUCH = 7,        // parent older than child
    CHK_PIN = 8,          // parent pinned less than child
    CHK_ORPHAN = 9,       // present key on no chain of the instance
};

__device__ __forceinline__ void chk_fail(const Params &P, int gi, int code) {
    if (atomicCAS(P.err, 0, DEV_E_INVARIANT) == 0) { P.err[1] = P.gbase + gi; P.err[2] = code; }
}

// one chain (keys[0..L)) on table T: every present key's depth and its parent relations
__device__ void chk_chain(const Params &P, const Table &T, int gi, const u64 *k0, int n0, const u64 *k1, int n1,
                          u32 *seen, int lane) {
    const int L = n0 + n1;
    for (int j = lane; j < L; j += 32) {
        const u64 key = j < n0 ? k0[j] : k1[j - n0];
        const int s = tab_find(T, key);
        if (s < 0) continue;
        atomicOr(seen + (s >> 5), 1u << (s & 31));
        const Meta m = load_meta(T.m + s);
        if (m.depth != j + 1) { chk_fail(P, gi, CHK_DEPTH); continue; }
        if (j == 0) continue;
        const u64 pk = j - 1 < n0 ? k0[j - 1] : k1[j - 1 - n0];
        const int ps = tab_find(T, pk);
        if (ps < 0) { chk_fail(P, gi, CHK_CLOSURE); continue; }
        const Meta pm = load_meta(T.m + ps);
        if (pm.depth != m.depth - 1) chk_fail(P, gi, CHK_DEPTH);
        if (pm.touch < m.touch) chk_fail(P, gi, CHK_TOUCH);
        if (pm.pin < m.pin) chk_fail(P, gi, CHK_PIN);
    }
}

// One warp per local instance. seen: (N << slog2) bits, zeroed by the caller.
// seg: API-inserted chains as (instance, arena offset, length) triples.
__global__ void check_invariants_kernel(Params P, i64 R, const i64 *seg, i64 nseg, u32 *seen) {
    const int gi = (int)((blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (gi >= P.N) return;
    const int g = P.gbase + gi;
    const Inst s = P.inst[gi];

    // reconcile (engine.py:248-258). Queue slots have generated == 0; a running
    // record's finish step v = join step + out - 1, so after step_idx steps it has
    // generated = out - 1 - (v - step_idx).
    {
        const QEnt *qb = P.qbuf + ((size_t)gi << P.qlog2);
        const int qmask = (1 << P.qlog2) - 1;
        i64 pend = 0, tot = 0, dc = 0;
        for (int j = lane; j < s.q; j += 32) {
            const QEnt &e = qb[(s.q_head + j) & qmask];
            pend += e.v;
            tot += e.in;
        }
        const REnt *rb = P.rbuf + (size_t)gi * (size_t)P.max_batch;
        for (int j = lane; j < s.r; j += 32) {
            const REnt &e = rb[j];
            const i64 gen = (i64)e.out - 1 - (e.v - s.step_idx);
            tot += e.in + gen;
            dc += e.in + gen;
        }
        pend = warp_sum(pend); tot = warp_sum(tot); dc = warp_sum(dc);
        if (lane == 0 && (pend != s.pend || tot != s.total || dc != s.dcs || s.q < 0 || s.r < 0 ||
                          s.r > P.max_batch))
            chk_fail(P, gi, CHK_AGG);
    }

    const Table T = table_of(P, gi);
    u32 *sn = seen + (((size_t)gi << P.slog2) >> 5);
    // chains of the requests routed here, then the API-inserted chains
    for (i64 r0 = 0; r0 < R; r0 += 32) {          // 32 requests per ballot, then their chains warp-wide
        u32 m = __ballot_sync(FULL, r0 + lane < R && P.chosen[r0 + lane] == g);
        while (m) {
            const i64 r = r0 + __ffs(m) - 1;
            m &= m - 1;
            const i64 a = P.blk_off[r], B = P.blk_off[r + 1] - a;
            const i64 oa = P.ooff[r], O = P.ooff[r + 1] - oa;
            chk_chain(P, T, gi, P.ckeys + a, (int)B, P.okeys + oa, (int)O, sn, lane);
        }
    }
    for (i64 i = 0; i < nseg; i++) {
        if (seg[3 * i] != gi) continue;
        chk_chain(P, T, gi, P.arena + seg[3 * i + 1], (int)seg[3 * i + 2], nullptr, 0, sn, lane);
    }
    __syncwarp();
    __threadfence_block();

    // every entry (kvcache.py:185-188), occupancy, orphans
    int cnt = 0;
    const u32 S = 1u << P.slog2;
    for (u32 i = lane; i < S; i += 32) {
        if (T.k[i] == T.empty) continue;
        cnt++;
        const Meta m = load_meta(T.m + i);
        if (m.depth < 1 || m.pin < 0) chk_fail(P, gi, CHK_ENTRY);
        if (!((sn[i >> 5] >> (i & 31)) & 1u)) chk_fail(P, gi, CHK_ORPHAN);
    }
    cnt = warp_sum(cnt);
    if (lane == 0) {
        if (cnt != s.occ) chk_fail(P, gi, CHK_OCC);
        if (P.cap > 0 && cnt > P.cap) chk_fail(P, gi, CHK_CAP);
    }
}

// Fault injection for the checker's own tests (rsim_debug_corrupt): 0 bumps the pin of the
// deepest entry of the instance's table (pin no longer covered by the parent), 1 breaks the
// running aggregates (total += 1), 2 ages the parent of the deepest entry.
__global__ void debug_corrupt_kernel(Params P, int gi, int what) {
    if (threadIdx.x != 0) return;
    if (what == 1) { P.inst[gi].total += 1; return; }
    const Table T = table_of(P, gi);
    int best = -1, bd = 0;
    for (u32 i = 0; i < (1u << P.slog2); i++)
        if (T.k[i] != T.empty && T.m[i].depth > bd) { bd = T.m[i].depth; best = (int)i; }
    if (best < 0) return;
    if (what == 0) { T.m[best].pin += 1; return; }
    // what == 2: the entry of depth bd - 1 with the largest touch is the parent candidate; age every
    // entry of that depth below the child's touch
    const i64 ct = T.m[best].touch;
    for (u32 i = 0; i < (1u << P.slog2); i++)
        if (T.k[i] != T.empty && T.m[i].depth == bd - 1) T.m[i].touch = ct - 1;
}
