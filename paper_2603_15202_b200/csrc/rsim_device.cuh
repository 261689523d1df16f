// rsim_device.cuh -- device-side data layout and warp primitives of librsim.
//
// Layout in HBM (one handle = one GPU's shard of instances):
//   trace (CSR, replicated):   arrival_us/in/out/rid [R], blk_off [R+1], blocks [sum B]
//   chain keys (K1 output):    ckeys (same CSR as blocks), okeys (output-block keys, CSR ooff)
//   per-request outputs:       chosen, hit_tokens, first_sched/first_token/finish, hit_blocks
//   per-instance engine state: Inst (loaded into shared memory for a persistent launch)
//   per-instance FIFO queue:   QEnt ring [Qcap]                 (engine.py:212)
//   per-instance running list: REnt [max_batch]                 (engine.py:213)
//   per-instance KV$ index:    open-addressing table, keys u64 [S] + Meta [S] (kvcache.py:47-60)
#pragma once
#include <stdint.h>

typedef long long i64;
typedef unsigned long long u64;
typedef unsigned int u32;

#define RSIM_NONE 0x7fffffffffffffffLL
#define RSIM_GOLDEN 0x9E3779B97F4A7C15ULL
#define RSIM_OUTPUT_SALT 0x0F0C0DEULL

// Error codes (match rsim_status in include/rsim.h)
#define DEV_E_CACHE_FULL 3
#define DEV_E_DUPLICATE 4
#define DEV_E_INVARIANT 5
#define DEV_E_QUEUE_OVERFLOW 7
#define DEV_E_TABLE_FULL 8
#define DEV_E_COMM 10
#define DEV_E_HISTORY_OVERFLOW 12
#define DEV_E_DETECTOR 13
#define DEV_E_RUNS_FULL 14

// A request on an instance: one 64-byte record used by the FIFO queue (v =
// pending prefill tokens) and the running list (v = finish step = join step +
// out - 1). It carries everything a step needs, so pops and finishes never
// reload per-request metadata.
struct __align__(16) Ent {
    i64 v;            // queue: pending prefill tokens; running: finish step
    i64 in;           // input tokens
    i64 a;            // offset of the request's prefix chain keys (ckeys)
    i64 oa;           // offset of its output-block keys (okeys)
    int req, flags;   // flags bit0: prefill scheduled at least once
    int out, B, L, hb;   // output tokens, prefix blocks, full chain length, admission hit blocks
    u64 kx;              // chain key at depth hb (the first key not cached at admission), 0 = unknown
};
typedef Ent QEnt;
typedef Ent REnt;

// Engine + router state of one instance. Live aggregates are the engine's
// truth (engine.py:219-222); v_* is the router-visible view that only syncs at
// step end (engine.py:224-246). next_finish caches min(finish_step) over the
// running list so steps without a finish never touch the list.
struct __align__(16) Inst {
    i64 next_step;    // next engine step start (RSIM_NONE = idle)     cluster.py:244-285 next_step[]
    i64 busy_until;   // engine.py:214
    i64 due;          // view sync due time (RSIM_NONE = none)         engine.py:227
    i64 pend, total, dcs;          // live pending / total / decode-context tokens
    i64 v_pend, v_total, v_dc;     // view
    i64 step_idx;     // steps executed so far
    i64 next_finish;  // min finish step among running (RSIM_NONE if none)
    i64 occ;          // KV$ occupancy (live chains)
    i64 r_head, r_tail, r_tailT;   // touch-run ring (finite capacity): positions and newest T
    i64 qcpos;        // queue ring index whose record qhead caches (-1: none)
    int r, q;         // live running / queued counts
    int v_r, v_q;     // view counts
    int q_head;       // queue ring head index
    int tabver;       // bumped whenever the KV$ key set may change (finish inserts / evictions):
                      // a probe made at version v stays valid while tabver == v
    int hhead, htail; // router-observable view history (engine.py:225, staleness > 0 only): a
                      // deque of (t, view) in the ring P.hring, live entries [hhead, htail);
                      // entry 0 is an implicit (-inf, zero view), so the deque is never empty
    Ent qhead;        // copy of the FIFO head record (valid while qcpos == q_head): the step that
                      // prefills a lone queued request reads it from shared memory, not L2
};
static_assert(sizeof(Inst) == 224, "Inst layout");

// one view-history entry (engine.py:225 history item): 32 B
struct __align__(16) HEnt { i64 t, pend, total; int r, q; };


__device__ __forceinline__ Ent shfl_ent(const Ent &e, int src) {
    Ent r;
    const u64 *p = reinterpret_cast<const u64 *>(&e);
    u64 *q = reinterpret_cast<u64 *>(&r);
#pragma unroll
    for (int i = 0; i < 8; i++) q[i] = __shfl_sync(0xffffffffu, p[i], src);
    return r;
}

struct Meta { i64 touch; int depth; int pin; };       // kvcache.py:34-41 (parent implied by the chain)

struct Params {
    // trace (device)
    const i64 *arrival, *in_tok, *out_tok, *blk_off, *ooff;
    const u64 *rid, *ckeys, *okeys;
    // per-request outputs / state
    int *hit_blocks, *chosen;
    i64 *hit_tokens, *first_sched, *first_token, *finish, *route_bs, *dec_ns;
    // cluster shape
    int N, C, W, ipw, per_cta;
    // model
    int bs, policy, kv_ind, bal_ind, debug;
    i64 cap, chunk, max_batch;
    double pb, pt, db, ds, dcc, qw;
    double kvw, bsn; i64 range_thr;   // linear weight / fixed normaliser, filter range threshold
    // instance state
    Inst *inst;
    QEnt *qbuf; int qlog2;
    REnt *rbuf;
    u64 *tkeys; Meta *tmeta; int slog2; i64 max_occ; u64 empty;
    // control
    u64 *tie;      // [2] = lo, hi of the TieBreaker counter
    int *err;      // [0] = first error code, [1] = instance, [2..3] info
    i64 *log; i64 log_cap; u64 *log_n;
    double *scores;   // optional per-instance scores of a route_one call
    u64 *ctr;         // [0] algorithmic probe bytes, [1] engine steps, [2] evictions
    struct Run *runs; int rlog2;   // per-instance touch-run rings (rsim_lru.cuh), null for infinite capacity
    const u64 *arena; // chain keys of API-inserted runs
    // multi-GPU shard: local instance i is global instance gbase + i
    int gbase, world, rank;
    u64 *mbox;        // this rank's mailbox [2 parity][8 ranks][4 words]
    u64 *peer[8];     // every rank's mailbox (peer-mapped), peer[rank] == mbox
    u64 epoch;        // run epoch, distinguishes mailbox contents of successive replays
    i64 timeout_ns;
    // diagnostics: per (decision, warp) phase record, 8 x u16 (rsim_phase_records); null = off
    unsigned short *crit; i64 crit_cap;
    i64 stal;         // router staleness in us (cluster.py:77); 0 = the live view
    HEnt *hring; int hlog2;            // per-instance view-history rings (staleness > 0)
    // prefix-hotspot detector (rsim_detector.cuh; single-CTA replay), dtid == nullptr: off
    const int *dtid;                   // [R] class track of each request (dense, by first arrival)
    const int *dtw; const i64 *dtex; const u64 *dtkey;   // [T] exemplar length / chain-key offset / class key
    struct DTrack *dtr;                // [T] track state
    i64 *dbk, *dtot, *dglob;           // buckets [T][BC][3], totals [BC][2], scalars (DG_*)
    i64 *drows; i64 drows_cap;         // emitted DetectorRows, 7 words each
    double dwin, dmult; i64 dwin_i, dcool;
    int dT, dtopk, dforce, dmean, dbclog2;
    int dTs;                           // track stride of the per-CTA bucket rings (>= dT)
    int dsm;                           // 1: the replay keeps tracks in shared memory
    i64 *ddbg;                         // diagnostics: 8 words per decision (rsim_detector_debug), null = off
    // simulate policy (policies.py:142-157, engine.py:419-460): the sim cost model and per-warp scratch
    double spb, spt, sdb, sds, sdc;
    int4 *simj;                        // [C*W][Qcap] (start step, last step, ctx at start, -) of joined requests
    // small shards: this CTA's running lists live in shared memory during a launch (byte offset of
    // the region in dynamic shared memory; 0 = global rbuf)
    int rsm_off;
    // one extra CTA (rank C of the cluster) decides every decision alone and broadcasts it
    // (replay_kernel, non-extended kernel): the instance CTAs' control warps only stage requests
    int central;
    // route() API: instances (global-id bitmap) already holding the routed request id -- a decision
    // for one of them raises DuplicateRequestError after the tie-break (engine.py:266-267); null = none
    const u32 *dupmask;
};

// running list of instance gi: shared memory (a launch of a small shard) or HBM
extern __shared__ __align__(16) unsigned char smem[];
__device__ __forceinline__ REnt *rlist(const Params &P, int gi) {
    if (P.rsm_off) return reinterpret_cast<REnt *>(smem + P.rsm_off) + (size_t)(gi % P.per_cta) * (size_t)P.max_batch;
    return P.rbuf + (size_t)gi * (size_t)P.max_batch;
}

// ---------------- hashing (hashing.py:15-25) ----------------
__device__ __forceinline__ u64 splitmix64(u64 z) {
    z += RSIM_GOLDEN;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__device__ __forceinline__ u64 combine64(u64 acc, u64 v) { return splitmix64(acc ^ v); }

// table home slot: Fibonacci hashing of the (already mixed) chain key
__device__ __forceinline__ u32 tab_home(u64 key, int slog2) {
    return (u32)((key * 0x9E3779B97F4A7C15ULL) >> (64 - slog2));
}

// ---------------- warp helpers ----------------
#define FULL 0xffffffffu
__device__ __forceinline__ u32 lanemask_lt() { u32 m; asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m)); return m; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}
__device__ __forceinline__ i64 warp_min_i64(i64 v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) { i64 w = __shfl_xor_sync(FULL, v, o); v = w < v ? w : v; }
    return v;
}
__device__ __forceinline__ i64 warp_max_i64(i64 v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) { i64 w = __shfl_xor_sync(FULL, v, o); v = w > v ? w : v; }
    return v;
}
__device__ __forceinline__ u64 warp_min_u64(u64 v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) { u64 w = __shfl_xor_sync(FULL, v, o); v = w < v ? w : v; }
    return v;
}
template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { T w = __shfl_up_sync(FULL, v, o); if (lane >= o) v += w; }
    return v;
}
// position of the k-th (0-based) set bit of m
// warp-wide form (m, k uniform across the warp): one popc + ballot instead of a k-step loop
__device__ __forceinline__ int nth_set_bit_warp(u32 m, int k, int lane) {
    const bool hit = ((m >> lane) & 1u) && __popc(m & lanemask_lt()) == k;
    return __ffs(__ballot_sync(FULL, hit)) - 1;
}
__device__ __forceinline__ int nth_set_bit(u32 m, int k) {
    for (int i = 0; i < k; i++) m &= m - 1;
    return __ffs(m) - 1;
}

__device__ __forceinline__ u64 ldcg_u64(const u64 *p) { return __ldcg(p); }

// ---------------- view history (staleness > 0) ----------------
// Drop the entries no snapshot with a cutoff >= `cutoff` can see (indicators.py:51-53):
// advance hhead while entry hhead + 1 exists and is at or before the cutoff.
__device__ __noinline__ void hist_make_room(const Params &P, Inst &s, int gi, i64 cutoff) {
    const HEnt *ring = P.hring + ((size_t)gi << P.hlog2);
    const int mask = (1 << P.hlog2) - 1;
    int hh = s.hhead;
    while (hh + 1 < s.htail && ring[(hh + 1) & mask].t <= cutoff) hh++;
    s.hhead = hh;
}
// history.append((t, view)) of instance gi (engine.py:245, 286); view = the v_* fields.
// now: the current simulated time -- no later snapshot has a cutoff below now - staleness.
__device__ __noinline__ void hist_append(const Params &P, Inst &s, int gi, i64 t, i64 now) {
    const int j = s.htail;
    if (j - s.hhead >= (1 << P.hlog2)) {             // full: drop what no later snapshot can see
        hist_make_room(P, s, gi, now - P.stal);
        if (j - s.hhead >= (1 << P.hlog2)) { atomicCAS(P.err, 0, DEV_E_HISTORY_OVERFLOW); return; }
    }
    HEnt e;
    e.t = t; e.pend = s.v_pend; e.total = s.v_total; e.r = s.v_r; e.q = s.v_q;
    P.hring[((size_t)gi << P.hlog2) + (j & ((1 << P.hlog2) - 1))] = e;
    s.htail = j + 1;
}

// Shared-memory cache of one instance's history head (extended kernel, staleness > 0):
// the view of entry hidx and the time of entry ntidx = hidx + 1 (-1: not cached).
struct __align__(16) HistHead { i64 pend, total, nt; int r, q, hidx, ntidx; };

// snapshot(now, staleness) of instance gi (indicators.py:36-65), after the caller's
// flush: pop, then the head is the latest entry at or before the cutoff (times are
// monotone and cutoffs never decrease). Leaves the stale view in c.
__device__ __forceinline__ void hist_snapshot(const Params &P, Inst &s, HistHead &c, int gi, i64 cutoff) {
    const HEnt *ring = P.hring + ((size_t)gi << P.hlog2);
    const int mask = (1 << P.hlog2) - 1;
    int hh = s.hhead;
    const int ht = s.htail;
    i64 nt = RSIM_NONE;
    if (hh + 1 < ht) nt = c.ntidx == hh + 1 ? c.nt : ring[(hh + 1) & mask].t;
    while (nt <= cutoff) {
        hh++;
        nt = hh + 1 < ht ? ring[(hh + 1) & mask].t : RSIM_NONE;
    }
    s.hhead = hh;
    if (c.hidx != hh) {
        if (hh == 0) { c.r = 0; c.q = 0; c.pend = 0; c.total = 0; }
        else { const HEnt e = ring[hh & mask]; c.r = e.r; c.q = e.q; c.pend = e.pend; c.total = e.total; }
        c.hidx = hh;
    }
    c.nt = nt; c.ntidx = hh + 1 < ht ? hh + 1 : -1;
}
