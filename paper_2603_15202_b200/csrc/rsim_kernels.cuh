// rsim_kernels.cuh -- the kernels of librsim.
//
//   k1_chain_keys    K1: prefix-chain keys + output-block keys for a request range
//   replay_kernel    K2-K4 fused persistent replay: per decision, drain engine
//                    steps (K4), probe + score every instance (K2), reduce to
//                    the rotating-tie-break argmin across the CTA cluster (K2),
//                    enqueue on the winner (K3)
//   probe_batch      what-if probe of many requests x all instances (no commits)
//   cache_op_kernel  single-instance PrefixCache operations for the API
#pragma once
#include "rsim_engine.cuh"
#include "rsim_detector.cuh"

// ---------------------------------------------------------------- K1
// One thread per request: the chain is sequential per request (splitmix64 is not
// associative, hashing.py:36-47), so every lane folds its own request's blocks
// at once, a full 32-B sector (4 keys) per iteration with the next sector's load
// in flight; keys go out as full-sector stores. Output-block keys extend the
// chain with stable_key(0x0F0C0DE, rid, idx) (engine.py:363-372).
#define K1_WARPS 8
__device__ __forceinline__ void k1_fold(u64 &acc, u64 v, u64 empty, bool &bad) {
    acc = combine64(acc, v);
    bad |= (acc == empty);
}
__global__ void __launch_bounds__(32 * K1_WARPS)
k1_chain_keys(const i64 *__restrict__ blk_off, const u64 *__restrict__ blocks, u64 *__restrict__ ckeys,
              const i64 *__restrict__ ooff, u64 *__restrict__ okeys, const u64 *__restrict__ rid,
              i64 r0, i64 r1, u64 empty, int *flag) {
    const i64 r = r0 + (i64)blockIdx.x * blockDim.x + threadIdx.x;
    bool bad = false;
    if (r < r1) {
        const i64 a = blk_off[r], b = blk_off[r + 1];
        u64 acc = RSIM_GOLDEN;
        i64 j = a;
        for (; j < b && (j & 3); j++) { k1_fold(acc, __ldcs(blocks + j), empty, bad); __stcs(ckeys + j, acc); }
        if (j + 4 <= b) {
            const ulonglong2 *src = reinterpret_cast<const ulonglong2 *>(blocks + j);
            ulonglong2 *dst = reinterpret_cast<ulonglong2 *>(ckeys + j);
            ulonglong2 x0 = __ldcs(src), x1 = __ldcs(src + 1);
            const i64 nq = (b - j) >> 2;
            for (i64 q = 0; q < nq; q++) {
                ulonglong2 n0 = x0, n1 = x1;
                if (q + 1 < nq) { n0 = __ldcs(src + 2 * q + 2); n1 = __ldcs(src + 2 * q + 3); }
                u64 k0 = acc, k1, k2, k3;
                k1_fold(k0, x0.x, empty, bad);
                k1 = k0; k1_fold(k1, x0.y, empty, bad);
                k2 = k1; k1_fold(k2, x1.x, empty, bad);
                k3 = k2; k1_fold(k3, x1.y, empty, bad);
                acc = k3;
                __stcs(dst + 2 * q, make_ulonglong2(k0, k1));
                __stcs(dst + 2 * q + 1, make_ulonglong2(k2, k3));
                x0 = n0; x1 = n1;
            }
            j += nq << 2;
        }
        for (; j < b; j++) { k1_fold(acc, __ldcs(blocks + j), empty, bad); __stcs(ckeys + j, acc); }
        const i64 o0 = ooff[r], o1 = ooff[r + 1];
        const u64 salt = combine64(combine64(RSIM_GOLDEN, RSIM_OUTPUT_SALT), rid[r]);
        for (i64 i = o0; i < o1; i++) {
            k1_fold(acc, combine64(salt, (u64)(i - o0)), empty, bad);
            okeys[i] = acc;
        }
    }
    if (__any_sync(FULL, bad) && (threadIdx.x & 31) == 0) atomicExch(flag, 1);
}

// ---------------------------------------------------------------- cluster PTX
__device__ __forceinline__ u32 cluster_ctarank() { u32 r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ u32 smem_addr(const void *p) { return (u32)__cvta_generic_to_shared(p); }
// ---- mbarrier + st.async: the cross-CTA partial exchange (no global-memory fence involved)
__device__ __forceinline__ void mbar_init(u64 *mb, u32 count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_addr(mb)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect(u64 *mb, u32 bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.release.cta.shared::cta.b64 st, [%0], %1;\n\t}"
                 :: "r"(smem_addr(mb)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(u64 *mb) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.release.cta.shared::cta.b64 st, [%0];\n\t}"
                 :: "r"(smem_addr(mb)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(u64 *mb, u32 parity) {
    u32 ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_addr(mb)), "r"(parity) : "memory");
    return ok != 0;
}
// 16-byte store into CTA `rank`'s shared memory that completes 16 tx-bytes on its mbarrier
__device__ __forceinline__ void st_async_16(const void *local_dst, const u64 *local_mb, u32 rank, u64 a, u64 b) {
    u32 rd, rm;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rd) : "r"(smem_addr(local_dst)), "r"(rank));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rm) : "r"(smem_addr(local_mb)), "r"(rank));
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.u64 [%0], {%1, %2}, [%3];"
                 :: "r"(rd), "l"(a), "l"(b), "r"(rm) : "memory");
}
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ void st_cluster_u64(u32 local_addr, u32 rank, u64 v) {
    u32 remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_addr), "r"(rank));
    asm volatile("st.shared::cluster.u64 [%0], %1;" :: "r"(remote), "l"(v) : "memory");
}

__device__ __forceinline__ void st_release_sys(u64 *p, u64 v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(u64 *p, u64 v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u64 ld_acquire_sys(const u64 *p) {
    u64 v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ u64 ld_relaxed_sys(const u64 *p) {
    u64 v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// explicit shared-space loads for pointers the compiler cannot prove to be shared
// (a generic LD to shared memory takes the L1TEX path and a long scoreboard)
__device__ __forceinline__ ulonglong2 lds_v2u64(const void *p) {
    ulonglong2 v;
    asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "r"(smem_addr(p)));
    return v;
}
__device__ __forceinline__ u64 lds_u64(const void *p) {
    u64 v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(smem_addr(p)));
    return v;
}
__device__ __forceinline__ u32 lds_u32(const void *p) {
    u32 v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_addr(p)));
    return v;
}
__device__ __forceinline__ u64 globaltimer() { u64 t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

struct __align__(16) Part { u64 minb; u32 cnt; u32 err; };

// ---------------------------------------------------------------- score
// Policy scores (policies.py:104-139) as IEEE doubles, bit-exact with
// CPython's float arithmetic (each op rounded to nearest, no contraction).
__device__ __forceinline__ double score_of(const Params &P, int v_r, int v_q, i64 v_pend, i64 v_total, int h, i64 in,
                                           double bsn = 1.0) {
    const i64 bsz = (i64)v_r + v_q;
    if (P.policy == 0) {                                            // multiplicative
        i64 ht = (i64)h * P.bs; if (ht > in) ht = in;
        i64 nw = in - ht; if (nw < 1) nw = 1;
        double kv = P.kv_ind == 0 ? __ll2double_rn(v_pend + nw)
                                  : __dsub_rn(1.0, __ddiv_rn(__ll2double_rn(ht), __ll2double_rn(in)));
        i64 bal = P.bal_ind == 0 ? bsz : v_total;
        return __dmul_rn(kv, __ll2double_rn(bal > 1 ? bal : 1));
    } else if (P.policy == 1) {                                     // vllm
        return __dadd_rn(__dmul_rn(P.qw, (double)v_q), (double)v_r);
    } else if (P.policy == 3 || P.policy == 4) {
        i64 ht = (i64)h * P.bs; if (ht > in) ht = in;
        const double hr = __ddiv_rn(__ll2double_rn(ht), __ll2double_rn(in));   // Candidate.hit_ratio
        if (P.policy == 4) return __dsub_rn(1.0, hr);               // filter, hit branch (policies.py:183)
        double load = __ddiv_rn(__ll2double_rn(bsz), bsn);          // linear (policies.py:109-114)
        if (!(load < 1.0)) load = 1.0;
        return __dadd_rn(__dmul_rn(P.kvw, __dsub_rn(1.0, hr)), __dmul_rn(__dsub_rn(1.0, P.kvw), load));
    }
    return __ll2double_rn(bsz);                                     // least_bs
}

// enqueue on the winner (InstanceSim.enqueue, engine.py:262-289) + route bookkeeping
// The touch + pin of the hit chain is parked in F (run_touch_pin) and runs after
// this warp's next publish, or earlier before cache work on the same instance.
__device__ __forceinline__ void commit(const Params &P, Inst *sp, int gi, i64 k, int h, i64 t, const u64 *keys128,
                                       const int *slot0, i64 a, int B, i64 in, int out, i64 oa, int lane, int &werr,
                                       FinBuf &F, bool stale) {
    // scalar work on lane 0: a handful of shared-memory fields and one 64-B queue record
    int bad = 0;
    __syncwarp();
    if (lane == 0) {
        const int q = sp->q;
        if (q >= (1 << P.qlog2)) {
            bad = 1;
        } else {
            F.tpn = h > 0; F.tpgi = gi; F.tph = h; F.tpver = sp->tabver; F.tpa = a; F.tpt = t;
            F.tpkeys = keys128; F.tpsl = slot0; F.tpsp = sp;
            i64 ht = (i64)h * P.bs; if (ht > in) ht = in;
            i64 pending = in - ht; if (pending < 1) pending = 1;
            Ent e;
            e.v = pending; e.in = in; e.a = a; e.oa = oa;
            e.req = (int)k; e.flags = 0; e.out = out; e.B = B;
            e.L = B + (int)((out + P.bs - 1) / P.bs); e.hb = h;
            e.kx = (h < B && h < 128) ? keys128[h] : 0ULL;
            P.qbuf[((size_t)gi << P.qlog2) + ((sp->q_head + q) & ((1 << P.qlog2) - 1))] = e;
            if (q == 0) { sp->qhead = e; sp->qcpos = sp->q_head; }     // the new record is the head
            P.hit_blocks[k] = h;
            P.chosen[k] = P.gbase + gi;
            P.hit_tokens[k] = ht;
            P.route_bs[k] = (i64)q + 1 + sp->r;
            sp->q = q + 1; sp->pend += pending; sp->total += in;
            sp->v_q += 1; sp->v_pend += pending; sp->v_total += in;   // view moves incrementally (engine.py:284-285)
            if (stale) hist_append(P, *sp, gi, t, t);                      // engine.py:286
            if (sp->next_step == RSIM_NONE && sp->busy_until <= t) sp->next_step = t;   // cluster.py:284-285
        }
    }
    if (__shfl_sync(FULL, bad, 0)) werr = DEV_E_QUEUE_OVERFLOW;
    __syncwarp();
}

enum { MODE_REPLAY = 0, MODE_DRAIN = 1, MODE_ROUTE = 2, MODE_ENQUEUE = 3 };

// One decision's request, staged once per CTA in shared memory by the CTA's
// control warp, up to RSIM_SLOTS-1 decisions ahead (slot k % RSIM_SLOTS).
struct __align__(16) ReqStage {
    i64 t, a, in, oa;
    int B, out;
    int dtid, dw;       // detector: class track and exemplar length
    u64 keys[128];
    u32 home[128];      // table home slot of each key (all instances share slog2)
};
struct __align__(16) Dec {
    int owner_warp; int kk; int err; int pad;   // owner warp in this CTA (-1: another CTA), its tie index, error, branch
    int oflat, okk, r0, r1;                     // the owner as a flat cluster warp index, its tie index (every CTA)
};

// Per-warp hand-off state between the phases of a decision.
struct __align__(16) WarpBuf {
    int slot[2][2][128];   // [decision parity][instance 0/1][depth]: probe-found table slots of the
                           // warp's first two instances (the commit reuses them instead of a lookup)
    int hit[32];           // hit blocks of each of the warp's instances for the current decision
    int sph[32];           // probe-ahead: hit blocks for decision spk, made at table version spver
    int spver[32];
    i64 spk;               // decision the probe-ahead results belong to (-1: none)
    FinBuf fin;            // finishers of one engine step
    u64 c_bytes, c_steps;  // algorithmic probe bytes / engine steps of this warp
    int werr, fins;        // first device error seen by this warp; finisher batches run
    // detector mode (rsim_detector.cuh): read by the control warp for the chosen instance
    i64 prod[32];          // p_tokens * max(bs, 1) of each instance (detector.py:312-316)
    int bsv[32];           // snapshot batch size
    u32 tm[6];             // tied-instance masks per argmin branch (policy, filter bs, holders excluded, least bs,
                           // filter bs among non-holders)
    __align__(16) unsigned char ecs[RSIM_DLMAX];   // holder counts of the listed tracks among this warp's instances
};

// counter mod T for the 128-bit TieBreaker counter (hi:lo) without a 128-bit
// division: Horner over 32-bit limbs, each step a 64-by-32 remainder.
__device__ __forceinline__ u32 mod_counter(u64 lo, u64 hi, u32 T) {
    u64 r = 0;
    if (hi) {
        r = ((u64)(u32)(hi >> 32)) % T;
        r = ((r << 32) | (u32)hi) % T;
    }
    r = ((r << 32) | (u32)(lo >> 32)) % T;
    r = ((r << 32) | (u32)lo) % T;
    return (u32)r;
}

#define RSIM_SLOTS 8            // request staging ring depth
#define RSIM_MBOX_W 8           // u64 words per (parity, rank) mailbox slot (filter: both branches + range)
#ifndef RSIM_DECODE_RUNS
// runs of pure decode steps in registers: 0 off, 1 every drain, 2 the drains off the critical path
// only. A/B on one B200 (us/decision, off / 1 / 2): api64 4.72 / 4.88 / 4.82, chat1024 6.61 /
// 6.75 / 6.67, agent256 19.37 / 18.32 / 18.95, adv64 7.96 / 8.20 / 7.97 -- the end-of-trace drain
// launch halves (chat1024 0.87 -> 0.45 ms) but the added code costs the replay loop more than
// the runs save on the headline shapes: off by default (profiles/r2_ab/ab_dr2.txt)
#define RSIM_DECODE_RUNS 0
#endif
#define RSIM_MAX_WARPS 8        // instance warps per CTA (+1 control warp)
#define RSIM_LEAN_WARPS 7       // up to 7 instance warps: 8 warps per CTA = 2 per SM sub-partition,
                                // which lifts the register budget from 168 to 255 per thread

// ---- control warp: stage decision k's request (scalars + first 128 chain keys)
__device__ __noinline__ void stage_request(const Params &P, ReqStage &R, i64 k, int mode, i64 until, int lane) {
    const i64 a = P.blk_off[k], e = P.blk_off[k + 1];
    const i64 t = (mode == MODE_REPLAY) ? P.arrival[k] : until;
    const i64 in = P.in_tok[k], oa = P.ooff[k], out = P.out_tok[k];
    const int B = (int)(e - a);
    u64 kk[4];
#pragma unroll
    for (int q = 0; q < 4; q++) kk[q] = (32 * q + lane < B) ? __ldcg(P.ckeys + a + 32 * q + lane) : 0;
#pragma unroll
    for (int q = 0; q < 4; q++)
        if (32 * q + lane < B) { R.keys[32 * q + lane] = kk[q]; R.home[32 * q + lane] = tab_home(kk[q], P.slog2); }
    if (lane == 0) { R.t = t; R.a = a; R.in = in; R.oa = oa; R.B = B; R.out = (int)out; }
    if (P.dtid != nullptr && mode != MODE_ENQUEUE && lane == 0) { R.dtid = P.dtid[k]; R.dw = P.dtw[R.dtid]; }
}

// ---- drain: advance instances [l0, l0+n) of this warp through steps starting before `until`
//      (cluster.py:250-273); skip_mask marks instances that must not move yet. The check is
//      inline; the (noinline) step function is only called when a step is due.
template <bool STALE, bool RUNS = (RSIM_DECODE_RUNS == 1)>
__device__ __forceinline__ void drain_phase(const Params &P, Inst *st, int base, int l0, int n, i64 until,
                                            u32 skip_mask, int lane, WarpBuf &WB, Defer *df = nullptr) {
    u32 due = __ballot_sync(FULL, lane < n && !((skip_mask >> lane) & 1u) && st[l0 + lane].next_step < until);
    while (due) {                                       // ascending instance order
        const int s = __ffs(due) - 1;
        due &= due - 1;
        Inst *sp = st + l0 + s;
        u64 steps = 0;
        while (sp->next_step < until && !WB.werr) {
#if RSIM_DECODE_RUNS
            if (RUNS && !(STALE && P.stal > 0) && sp->q == 0 && sp->r > 0 && sp->next_finish != sp->step_idx) {
                // a run of pure decode steps (no queue to plan, no finish before the next finish
                // step): inst_step_body's fast path step after step, on lane-uniform registers, with
                // one write-back -- each step flushes the view at its start (engine.py:293), adds
                // one token per running request and ends after decode_cost_us (engine.py:333-352)
                const int nd = sp->r;
                const i64 nf = sp->next_finish;
                i64 t = sp->next_step, si = sp->step_idx, dcs = sp->dcs, total = sp->total;
                bool fl = sp->due <= t, any = false;
                i64 fv_total = 0, fv_dc = 0, n = 0;
                const int gi = base + l0 + s;
                do {
                    if (fl) { fv_total = total; fv_dc = dcs; any = true; }
                    const i64 end = t + decode_cost_us(P, nd, dcs);
                    log_step(P, WB.fin, gi, t, end, 0, (i64)nd, si, lane);
                    total += nd; dcs += nd; si++; t = end; n++;
                    fl = true;                                   // (due = this end from here on)
                } while (t < until && si != nf);
                __syncwarp();
                if (lane == 0) {
                    if (any) { sp->v_r = nd; sp->v_q = 0; sp->v_pend = sp->pend; sp->v_total = fv_total; sp->v_dc = fv_dc; }
                    sp->total = total; sp->dcs = dcs; sp->step_idx = si;
                    sp->busy_until = t; sp->due = t; sp->next_step = t;
                }
                __syncwarp();
                steps += (u64)n;
                continue;
            }
#endif
            if (STALE && P.stal > 0 && sp->due <= sp->next_step) {   // the step's flush (engine.py:293), recorded
                __syncwarp();
                if (lane == 0) flush_view_hist(P, *sp, base + l0 + s, sp->next_step);
                __syncwarp();
            }
            steps += inst_step(P, sp, base + l0 + s, s, lane, &WB.werr, WB.fin, df);
        }
        if (lane == 0) WB.c_steps += steps;
    }
}

// ---- longest present prefix beyond the first 128 depths for up to 4 instances at once
// (instances gi0 + q for the bits q of dm), all of whose first 128 depths are present.
// Presence is monotone in depth (prefix closure, kvcache.py:4-7), so lane li first probes depth
// 128 + li*S (S = ceil((B-128)/32)); the first missing lane brackets the boundary within S
// depths, which a second lookup of <= 64 depths (two per lane) pins. The stage-1 keys are the
// request's and shared by all instances: two round trips of table loads for all four
// instances instead of ~3 rounds of (key load, table load) per instance (deep_match). Longer
// prompts (S > 65) take deep_match.
__device__ __noinline__ void deep_hits(const Params &P, int gi0, u32 dm, const u64 *keys, int B, int lane, int *hout) {
    const int span = B - 128, S = (span + 31) / 32;
    if (S > 65) {
        for (u32 b = dm; b; b &= b - 1) {
            const int q = __ffs(b) - 1;
            const int h = deep_match(table_of(P, gi0 + q), keys, B, lane);
            if (lane == 0) hout[q] = min(h, B);
        }
        __syncwarp();
        return;
    }
    const int d1 = 128 + lane * S;
    const bool v1 = d1 < B;
    const u64 k1 = v1 ? keys[d1] : 0ULL;
    ulonglong2 pr[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const Table T = table_of(P, gi0 + (((dm >> q) & 1u) ? q : 0));
        pr[q] = (((dm >> q) & 1u) && v1) ? ld_pair(T, tab_home(k1, T.slog2)) : make_ulonglong2(0ULL, 0ULL);
    }
    int lo[4], cnt[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
        lo[q] = 128; cnt[q] = 0;
        if ((dm >> q) & 1u) {                                    // warp-uniform
            const Table T = table_of(P, gi0 + q);
            bool f = false, c = false;
            if (v1) eval_first(T, pr[q], tab_home(k1, T.slog2), k1, f, c);
            if (__any_sync(FULL, c) && c) {
                int stt;
                probe_rest(T, ((tab_home(k1, T.slog2) | 1u) + 1u) & T.mask, k1, stt);
                f = stt == 0;
            }
            const u32 bits = __ballot_sync(FULL, f);
            const int m = bits == FULL ? 32 : __ffs(~bits) - 1;  // lanes 0..m-1 present
            if (m > 0) {
                lo[q] = 128 + (m - 1) * S + 1;                  // depth 128+(m-1)S present
                cnt[q] = min(128 + m * S, B) - lo[q];            // depths lo..lo+cnt-1 unknown
            }
        }
    }
    u64 k2[4][2];
    ulonglong2 p2[4][2];
#pragma unroll
    for (int q = 0; q < 4; q++)
#pragma unroll
        for (int j = 0; j < 2; j++) {
            const bool v2 = ((dm >> q) & 1u) && 32 * j + lane < cnt[q];
            k2[q][j] = v2 ? keys[lo[q] + 32 * j + lane] : 0ULL;
        }
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const Table T = table_of(P, gi0 + (((dm >> q) & 1u) ? q : 0));
#pragma unroll
        for (int j = 0; j < 2; j++) {
            const bool v2 = ((dm >> q) & 1u) && 32 * j + lane < cnt[q];
            p2[q][j] = v2 ? ld_pair(T, tab_home(k2[q][j], T.slog2)) : make_ulonglong2(0ULL, 0ULL);
        }
    }
#pragma unroll
    for (int q = 0; q < 4; q++) {
        if ((dm >> q) & 1u) {                                    // warp-uniform
            const Table T = table_of(P, gi0 + q);
            int miss = 64;
#pragma unroll
            for (int j = 1; j >= 0; j--) {
                const bool v2 = 32 * j + lane < cnt[q];
                bool f = false, c = false;
                const u32 hm2 = tab_home(k2[q][j], T.slog2);
                if (v2) eval_first(T, p2[q][j], hm2, k2[q][j], f, c);
                if (__any_sync(FULL, c) && c) {
                    int stt;
                    probe_rest(T, ((hm2 | 1u) + 1u) & T.mask, k2[q][j], stt);
                    f = stt == 0;
                }
                const u32 mb = __ballot_sync(FULL, v2 && !f);
                if (mb) miss = 32 * j + __ffs(mb) - 1;
            }
            const int h = lo[q] + min(miss, cnt[q]);
            if (lane == 0) hout[q] = min(h, B);
        }
    }
    __syncwarp();
}

// ---- probe this warp's instances (cluster.py:106-128 -> kvcache.py:65-74): longest
// present prefix of request R in each instance's table, for instances not in
// `skip`. Short prompts are probed several instances at a time: the warp splits
// into G lane groups of LP = 32/G lanes, lane li of group g probing depths
// j*LP+li (j < 4) of instance s0+g, so one round trip and one instruction
// stream cover G instances. Hit blocks go to hout[s]; found slots of
// instances 0/1 to slot[s][depth].
// Out of line on purpose: a fresh register budget keeps the batch of loads in registers (inlined
// into the replay loop, ptxas spilled them and every load serialised on its spill store).
__device__ __noinline__ void probe_hits(const Params &P, int base, int l0, int n, const ReqStage &R, int mode,
                                        int target, u32 skip, int lane, int *hout, int (*slot)[128],
                                        bool diag = false) {
#ifdef RSIM_DIAG
    long long pt0 = clock64(), pt1 = 0, pt2 = 0;
#define PMARK(v) do { if (diag) v = clock64(); } while (0)
#else
#define PMARK(v) do { } while (0)
#endif
    const int B = R.B;
    const int Bc = min(B, 128);
    const int G = Bc <= 32 ? 4 : (Bc <= 64 ? 2 : 1);       // instances per round (warp-uniform)
    const int LP = 32 / G, DS = (Bc + LP - 1) / LP;         // lanes per instance, depth slots per lane
    const int g = lane / LP, li = lane - g * LP;
    const u32 gmask = LP == 32 ? FULL : ((1u << LP) - 1u);
    u32 need = (n >= 32 ? FULL : ((1u << n) - 1u)) & ~skip;
    if (mode == MODE_ENQUEUE) {
        const int tl = target - base - l0;
        need &= (tl >= 0 && tl < n) ? (1u << tl) : 0u;
    }
    if (need == 0) return;
    u64 kk[4];
    u32 hm[4];
    bool vd[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
        const int d = j * LP + li;
        vd[j] = j < DS && d < B;
        kk[j] = vd[j] ? lds_u64(R.keys + d) : 0;
        hm[j] = vd[j] ? lds_u32(R.home + d) : 0;
    }
    // rounds of G instances, issued four rounds at a time: every load of a batch is in flight
    // before the first is evaluated (one memory round trip per 4 rounds, not per round)
    const int nr = (n + G - 1) / G;
    PMARK(pt1);
    for (int b0 = 0; b0 < nr; b0 += 4) {
        ulonglong2 pr[4][4];
        bool cd[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int s = (b0 + q) * G + g;
            cd[q] = b0 + q < nr && s < n && ((need >> s) & 1u);
            const Table T = table_of(P, base + l0 + (cd[q] ? s : 0));
#pragma unroll
            for (int j = 0; j < 4; j++)        // unconditional assignment keeps pr in registers
                pr[q][j] = (cd[q] && vd[j]) ? ld_pair(T, hm[j]) : make_ulonglong2(0ULL, 0ULL);
        }
        PMARK(pt2);
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int s0 = (b0 + q) * G;
            if (b0 + q < nr && ((need >> min(s0, 31)) & ((1u << G) - 1u)) != 0) {   // warp-uniform
            const int s = s0 + g;
            const bool cand = cd[q];
            const Table T = table_of(P, base + l0 + (s < n ? s : s0));
            u32 mk[4];
#pragma unroll
            for (int j = 0; j < 4; j++) {
                mk[j] = 0;
                if (j < DS) {
                    bool f = false, c = false;
                    if (cand && vd[j]) eval_first(T, pr[q][j], hm[j], kk[j], f, c);
                    int sl = -1;
                    if (__any_sync(FULL, c) && c) {          // rare: the home pair is full of other keys
                        int stt;
                        const u32 r = probe_rest(T, ((hm[j] | 1u) + 1u) & T.mask, kk[j], stt);
                        f = stt == 0;
                        if (f) sl = (int)r;
                    } else if (f) {
                        sl = (int)((hm[j] & 1u) == 0 && pr[q][j].x == kk[j] ? hm[j] : hm[j] | 1u);
                    }
                    if (cand && s < 2 && vd[j]) slot[s][j * LP + li] = sl;
                    mk[j] = __ballot_sync(FULL, f);
                }
            }
            // leading present depths of my group's instance
            int h = DS * LP;
            bool done = false;
#pragma unroll
            for (int j = 0; j < 4; j++) {
                if (j < DS) {
                    const u32 bits = (mk[j] >> (g * LP)) & gmask;
                    if (!done && bits != gmask) { h = j * LP + __ffs(~bits) - 1; done = true; }
                }
            }
            h = min(h, B);
            if (cand && li == 0) hout[s] = h;                    // 128 of > 128: refined below
            }
        }
        if (G == 1 && B > 128) {                                 // warp-uniform
            __syncwarp();
            u32 dm = 0;
#pragma unroll
            for (int q = 0; q < 4; q++)
                if (b0 + q < nr && ((need >> min(b0 + q, 31)) & 1u) && hout[b0 + q] == 128) dm |= 1u << q;
            if (dm) deep_hits(P, base + l0 + b0, dm, P.ckeys + R.a, B, lane, hout + b0);
        }
    }
#ifdef RSIM_DIAG
    if (diag && lane == 0) {
        const long long pt3 = clock64();
        atomicAdd(P.ctr + 32, (u64)(pt1 - pt0)); atomicAdd(P.ctr + 33, (u64)(pt2 - pt1));
        atomicAdd(P.ctr + 34, (u64)(pt3 - pt2));
    }
#endif
#undef PMARK
    __syncwarp();
}

// ---- two-stage probe for warps that own several instances (prompts of <= 128 blocks). The
// dense probe costs B lookups per instance and the SM's load unit handles ~1 line per cycle,
// so with 10 instances per warp the probe-ahead was throughput-bound. Presence is monotone
// in depth (prefix closure, kvcache.py:4-7): one lookup per lane at stride S = ceil(B/LP)
// brackets the first miss within S depths, a second lookup of at most S-1 depths pins it:
// <= LP + S - 1 lookups per instance. Both stages batch up to 8 rounds of G instances.
__device__ __noinline__ void probe_hits_sparse(const Params &P, int base, int l0, int n, const ReqStage &R, int mode,
                                               int target, u32 skip, int lane, int *hout) {
    const int B = R.B;
    const int G = B <= 32 ? 4 : (B <= 64 ? 2 : 1);
    const int LP = 32 / G, S = (B + LP - 1) / LP;
    const int g = lane / LP, li = lane - g * LP;
    const u32 gmask = LP == 32 ? FULL : ((1u << LP) - 1u);
    u32 need = (n >= 32 ? FULL : ((1u << n) - 1u)) & ~skip;
    if (mode == MODE_ENQUEUE) {
        const int tl = target - base - l0;
        need &= (tl >= 0 && tl < n) ? (1u << tl) : 0u;
    }
    if (need == 0) return;
    const int d1 = li * S;
    const bool v1 = d1 < B;
    const u64 k1 = v1 ? lds_u64(R.keys + d1) : 0ULL;
    const u32 h1 = v1 ? lds_u32(R.home + d1) : 0u;
    const int nr = (n + G - 1) / G;
    for (int b0 = 0; b0 < nr; b0 += 8) {
        ulonglong2 pr[8];
        bool cd[8];
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const int s = (b0 + q) * G + g;
            cd[q] = b0 + q < nr && s < n && ((need >> s) & 1u);
            const Table T = table_of(P, base + l0 + (cd[q] ? s : 0));
            pr[q] = (cd[q] && v1) ? ld_pair(T, h1) : make_ulonglong2(0ULL, 0ULL);
        }
        // stage 1: first miss lane m of each group -> segment of candidate depths
        int lo[8], cnt[8];
#pragma unroll
        for (int q = 0; q < 8; q++) {
            lo[q] = 0; cnt[q] = 0;
            if (b0 + q < nr) {                                            // warp-uniform
                const int s = (b0 + q) * G + g;
                const Table T = table_of(P, base + l0 + (cd[q] ? s : 0));
                bool f = false, c = false;
                if (cd[q] && v1) eval_first(T, pr[q], h1, k1, f, c);
                if (__any_sync(FULL, c) && c) {
                    int stt;
                    probe_rest(T, ((h1 | 1u) + 1u) & T.mask, k1, stt);
                    f = stt == 0;
                }
                const u32 bits = (__ballot_sync(FULL, f) >> (g * LP)) & gmask;
                const int m = bits == gmask ? LP : __ffs(~bits) - 1;   // lanes 0..m-1 present
                lo[q] = m == 0 ? 0 : (m - 1) * S + 1;                     // depth (m-1)*S present
                cnt[q] = m == 0 ? 0 : min(m * S, B) - lo[q];              // depths lo..lo+cnt-1 unknown
            }
        }
        ulonglong2 p2[8];
        u64 k2[8];
        u32 hh2[8];
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const int s = (b0 + q) * G + g;
            const bool v2 = cd[q] && li < cnt[q];
            const int d2 = lo[q] + li;
            k2[q] = v2 ? lds_u64(R.keys + d2) : 0ULL;
            hh2[q] = v2 ? lds_u32(R.home + d2) : 0u;
            const Table T = table_of(P, base + l0 + (cd[q] ? s : 0));
            p2[q] = v2 ? ld_pair(T, hh2[q]) : make_ulonglong2(0ULL, 0ULL);
        }
#pragma unroll
        for (int q = 0; q < 8; q++) {
            if (b0 + q < nr) {                                            // warp-uniform
                const int s = (b0 + q) * G + g;
                const bool v2 = cd[q] && li < cnt[q];
                const Table T = table_of(P, base + l0 + (cd[q] ? s : 0));
                bool f = false, c = false;
                if (v2) eval_first(T, p2[q], hh2[q], k2[q], f, c);
                if (__any_sync(FULL, c) && c) {
                    int stt;
                    probe_rest(T, ((hh2[q] | 1u) + 1u) & T.mask, k2[q], stt);
                    f = stt == 0;
                }
                const u32 bits = (__ballot_sync(FULL, f) >> (g * LP)) & gmask;
                const u32 cm = cnt[q] >= LP ? gmask : ((1u << cnt[q]) - 1u);
                const int h = lo[q] + ((bits & cm) == cm ? cnt[q] : __ffs(~bits) - 1);
                if (cd[q] && li == 0) hout[s] = min(h, B);
            }
        }
    }
    __syncwarp();
}

// ---- score this warp's instances from their hit blocks (policies.py:117-139); lane s
// handles instance s and returns its score bits (~0 = not a candidate).
__device__ __forceinline__ u64 score_phase(const Params &P, Inst *st, int base, int l0, int n, const ReqStage &R,
                                           int mode, int target, int lane, WarpBuf &WB, u64 &bits_bs, bool filter,
                                           double bsn, bool stale, const HistHead *hc, bool det = false,
                                           int4 *simj = nullptr) {
    const int gi = base + l0 + lane;
    const bool cand = lane < n && ((mode != MODE_ENQUEUE) || gi == target);
    u64 bits = ~0ULL;
    bits_bs = ~0ULL;                                   // filter: the batch-size branch (policies.py:181)
    u32 cb = 0;
    if (cand) {
        Inst *sp = st + l0 + lane;
        // snapshot() flushes every candidate (indicators.py:36-65): the view is the live state once due
        int vr, vq;
        i64 vp, vt;
        if (stale) {       // stale_snapshot() ran: the history head is the view as of t - staleness
            const HistHead &c = hc[l0 + lane];
            vr = c.r; vq = c.q; vp = c.pend; vt = c.total;
        } else {
            const bool fl = sp->due <= R.t;
            vr = fl ? sp->r : sp->v_r; vq = fl ? sp->q : sp->v_q;
            vp = fl ? sp->pend : sp->v_pend; vt = fl ? sp->total : sp->v_total;
            if (fl) { sp->v_r = vr; sp->v_q = vq; sp->v_pend = vp; sp->v_total = vt; sp->v_dc = sp->dcs; sp->due = RSIM_NONE; }
        }
        const int h = WB.hit[lane];
        const double sc = score_of(P, vr, vq, vp, vt, h, R.in, bsn);
        if (det) {                                     // Candidate.p_tokens * max(bs, 1), snapshot bs
            i64 ht = (i64)h * P.bs; if (ht > R.in) ht = R.in;
            i64 nw = R.in - ht; if (nw < 1) nw = 1;
            const i64 bsz = (i64)vr + vq;
            WB.prod[lane] = (vp + nw) * (bsz > 1 ? bsz : 1);
            WB.bsv[lane] = (int)bsz;
            if (mode == MODE_ROUTE && P.scores != nullptr) {   // route()'s RoutingDecision under a verdict
                P.scores[2 * P.N + gi] = __ll2double_rn(bsz);
                P.scores[3 * P.N + gi] = h >= R.dw ? 1.0 : 0.0;
                P.scores[4 * P.N + gi] = sc;
            }
        }
        bits = (u64)__double_as_longlong(sc);
        if (P.scores != nullptr) P.scores[gi] = sc;
        if (filter) {
            const double sb = __ll2double_rn((i64)vr + vq);
            bits_bs = (u64)__double_as_longlong(sb);
            if (P.scores != nullptr) P.scores[P.N + gi] = sb;
        }
        // one 8-B key compare per reference dict lookup + 16 B of view
        cb = 8u * (u32)min(h + 1, R.B) + 16u;
    }
    if (simj != nullptr) {     // simulate: float(estimate_first_token_us - now) (policies.py:142-157, 262-267)
        for (int s = 0; s < n; s++) {
            const int g = base + l0 + s;
            if (mode == MODE_ENQUEUE && g != target) continue;          // warp-uniform
            i64 ht = (i64)WB.hit[s] * P.bs; if (ht > R.in) ht = R.in;
            const i64 nw = R.in - ht;                                   // Candidate.new_prefill_tokens (>= 1 inside)
            const i64 ft = sim_first_token(P, st + l0 + s, g, R.t, nw, lane, simj);
            if (ft < 0 && lane == 0) atomicCAS(P.err, 0, DEV_E_INVARIANT);   // "TTFT replay did not converge"
            if (lane == s) {
                const double sc = __ll2double_rn(ft - R.t);
                bits = (u64)__double_as_longlong(sc);
                if (P.scores != nullptr) P.scores[g] = sc;
            }
        }
    }
    cb = __reduce_add_sync(FULL, cb);
    if (lane == 0) WB.c_bytes += cb;
    return bits;
}

// TieBreaker counter at decision time = c0 + ties, c0 the launch-start value: counter mod T
// is (c0 mod T + ties mod T) mod T with c0 mod T memoised per T (modtab, T < RSIM_MODTAB;
// 0xffffffff = not computed yet: a launch sees few distinct tie counts, and a one-decision
// route() launch should not pay for 2048 128-bit remainders up front). Called by the whole
// control warp with the same T, so every lane computes and stores the same value.
#define RSIM_MODTAB 2048
__device__ __forceinline__ u32 tie_index(u32 *modtab, u64 c0_lo, u64 c0_hi, u32 ties, u32 T) {
    if (T < RSIM_MODTAB) {
        u32 m = modtab[T];
        if (m == 0xffffffffu) { m = mod_counter(c0_lo, c0_hi, T); modtab[T] = m; }
        u32 r = m + ties % T;
        return r >= T ? r - T : r;
    }
    u64 lo = c0_lo + ties;
    return mod_counter(lo, c0_hi + (lo < c0_lo), T);
}

template <int NRT>      // rounds of 32 partials (CW <= 16 CTAs x 8 warps = 128: NRT <= 4)
__device__ __forceinline__ void decide_phase_n(const Params &P, const Part *part, int CW, int W, int cta, i64 k, int par,
                                             Dec &dec, u32 *modtab, u64 c0_lo, u64 c0_hi, u32 &ties, int lane,
                                             bool filter, const Part *det_branch = nullptr, int det_code = 0) {
    // round-major: lane holds flat partials r*32 + lane (conflict-free 16-byte loads); flat
    // order = ascending instance id
#ifdef RSIM_DIAG
    const bool dg = P.ctr != nullptr && cta == 0 && lane == 0;
    long long dt0 = clock64(), dt1 = 0, dt2 = 0, dt3 = 0;
#endif
    u64 pm[NRT];
    u32 pc[NRT];
    u64 mn = ~0ULL;
    u32 er = 0;
    const int NR = (CW + 31) >> 5;
    const Part *pp = part + par * 2 * CW;
    bool bs_branch = false;
    bool pre = false;                            // filter across ranks: the exchange already ran
    u64 pre_min = ~0ULL;
    u32 pre_T = 0u, pre_er = 0u;
    if (filter) {              // route_filter (policies.py:168-192): bs range over all candidates
        u64 bmn = ~0ULL;
        u32 bmx = 0;
#pragma unroll
        for (int r = 0; r < NRT; r++) {
            const int idx = r * 32 + lane;
            if (r < NR && idx < CW) {
                const ulonglong2 q = lds_v2u64(pp + CW + idx);
                bmn = min(bmn, q.x); bmx = max(bmx, (u32)(q.y >> 32));
            }
        }
        const u32 bh = __reduce_min_sync(FULL, (u32)(bmn >> 32));
        const u64 gb = ((u64)bh << 32) | __reduce_min_sync(FULL, (u32)(bmn >> 32) == bh ? (u32)bmn : ~0u);
        const i64 bs_lo = gb == ~0ULL ? 0 : (i64)__longlong_as_double((long long)gb);
        const i64 bs_hi = (i64)__reduce_max_sync(FULL, bmx);
        bs_branch = bs_hi - bs_lo > P.range_thr;
        if (P.world > 1) {
            // route_filter's range is over ALL candidates, i.e. every rank's: each rank sends both
            // branches' (min, tie count) with its range in one mailbox message, and every rank
            // picks the branch from the global range (then the winner as for one policy)
            u64 m0 = ~0ULL, m1 = ~0ULL;
            u32 e0 = 0u;
#pragma unroll
            for (int r = 0; r < NRT; r++) {
                const int idx = r * 32 + lane;
                if (r < NR && idx < CW) {
                    const ulonglong2 q0 = lds_v2u64(pp + idx), q1 = lds_v2u64(pp + CW + idx);
                    m0 = min(m0, q0.x); m1 = min(m1, q1.x); e0 |= (u32)(q0.y >> 32);
                }
            }
            const u64 g0 = warp_min_u64(m0), g1 = warp_min_u64(m1);
            u32 t0 = 0u, t1 = 0u;
#pragma unroll
            for (int r = 0; r < NRT; r++) {
                const int idx = r * 32 + lane;
                if (r < NR && idx < CW) {
                    const ulonglong2 q0 = lds_v2u64(pp + idx), q1 = lds_v2u64(pp + CW + idx);
                    t0 += q0.x == g0 ? (u32)q0.y : 0u; t1 += q1.x == g1 ? (u32)q1.y : 0u;
                }
            }
            t0 = __reduce_add_sync(FULL, t0); t1 = __reduce_add_sync(FULL, t1);
            e0 = __reduce_or_sync(FULL, e0);
            const u64 seq = (P.epoch << 40) | (u64)(k + 1);
            if (cta == 0 && lane < P.world) {
                u64 *slot = P.peer[lane] + (size_t)((par * 8 + P.rank) * RSIM_MBOX_W);
                st_relaxed_sys(slot + 0, g0);
                st_relaxed_sys(slot + 1, ((u64)e0 << 32) | t0);
                st_relaxed_sys(slot + 3, g1);
                st_relaxed_sys(slot + 4, (u64)t1);
                st_relaxed_sys(slot + 5, (u64)bs_lo);
                st_relaxed_sys(slot + 6, (u64)bs_hi);
                st_release_sys(slot + 2, seq);
            }
            u64 a0 = ~0ULL, a1 = ~0ULL;
            u32 c0 = 0u, c1 = 0u, re = 0u;
            i64 lo = INT64_MAX, hi = INT64_MIN;
            if (lane < P.world) {
                const u64 *slot = P.mbox + (size_t)((par * 8 + lane) * RSIM_MBOX_W);
                const u64 tt = globaltimer();
                while (ld_relaxed_sys(slot + 2) != seq) {
                    if ((i64)(globaltimer() - tt) > P.timeout_ns) { re = DEV_E_COMM; break; }
                }
                asm volatile("fence.acq_rel.sys;" ::: "memory");
                if (!re) {
                    a0 = ld_relaxed_sys(slot + 0);
                    const u64 ce = ld_relaxed_sys(slot + 1);
                    c0 = (u32)ce; re = (u32)(ce >> 32);
                    a1 = ld_relaxed_sys(slot + 3);
                    c1 = (u32)ld_relaxed_sys(slot + 4);
                    lo = (i64)ld_relaxed_sys(slot + 5);
                    hi = (i64)ld_relaxed_sys(slot + 6);
                }
            }
            lo = warp_min_i64(lo); hi = warp_max_i64(hi);
            bs_branch = hi - lo > P.range_thr;
            pre_min = bs_branch ? a1 : a0;
            pre_T = bs_branch ? c1 : c0;
            pre_er = re;
            pre = true;
        }
    }
#pragma unroll
    for (int r = 0; r < NRT; r++) {
        const int idx = r * 32 + lane;
        pm[r] = ~0ULL; pc[r] = 0;
        if (r < NR && idx < CW) {
            const ulonglong2 q = lds_v2u64(pp + idx);
            er |= (u32)(q.y >> 32);
            const ulonglong2 qs = det_branch ? lds_v2u64(det_branch + idx)
                                  : bs_branch ? lds_v2u64(pp + CW + idx) : q;   // the chosen branch
            pm[r] = qs.x; pc[r] = (u32)qs.y; mn = min(mn, qs.x);
        }
    }
    u32 cl = 0;                                   // largest tie count of any partial
#pragma unroll
    for (int r = 0; r < NRT; r++) cl = max(cl, pc[r]);
    // 64-bit min with two 32-bit redux ops
    const u32 hmin = __reduce_min_sync(FULL, (u32)(mn >> 32));
    const u32 cmax = __reduce_max_sync(FULL, cl);
    er = __reduce_or_sync(FULL, er);
    const u32 lmin = __reduce_min_sync(FULL, (u32)(mn >> 32) == hmin ? (u32)mn : 0xffffffffu);
    const u64 gmin = ((u64)hmin << 32) | lmin;
    // every partial holds at most one tie (one instance per warp, or no intra-warp ties):
    // the tied partials are ballot bits, the kk-th one is a bit position, no prefix scan
    const bool single = cmax <= 1;
    u32 tb[NRT];
    u32 lc = 0, T = 0;
#pragma unroll
    for (int r = 0; r < NRT; r++) {
        pc[r] = pm[r] == gmin ? pc[r] : 0u;
        lc += pc[r];
        tb[r] = (single && r < NR) ? __ballot_sync(FULL, pc[r] > 0) : 0u;
        T += __popc(tb[r]);
    }
    if (!single) T = __reduce_add_sync(FULL, lc);
#ifdef RSIM_DIAG
    dt1 = clock64();
#endif
    Dec d; d.owner_warp = -1; d.kk = 0; d.err = (int)er; d.pad = 0; d.oflat = -1; d.okk = 0; d.r0 = d.r1 = 0;
    u32 kk = 0;
    bool mine = true;
    u32 Tg = T;
    if (P.world > 1) {          // ---- one (min, tie count) partial per rank over peer-mapped mailboxes
        const u64 seq = (P.epoch << 40) | (u64)(k + 1);
        if (!pre && cta == 0 && lane < P.world) {
            u64 *slot = P.peer[lane] + (size_t)((par * 8 + P.rank) * RSIM_MBOX_W);
            st_relaxed_sys(slot + 0, gmin);
            st_relaxed_sys(slot + 1, ((u64)er << 32) | T);
            st_release_sys(slot + 2, seq);
        }
        u64 rmin = pre ? pre_min : ~0ULL;
        u32 rT = pre ? pre_T : 0u, rer = pre ? pre_er : 0u;
        if (!pre && lane < P.world) {
            const u64 *slot = P.mbox + (size_t)((par * 8 + lane) * RSIM_MBOX_W);
            const u64 t0 = globaltimer();
            // relaxed polls (an acquire load at sys scope flushes L1 on every iteration), one
            // acquire fence once the sequence word matches
            while (ld_relaxed_sys(slot + 2) != seq) {
                if ((i64)(globaltimer() - t0) > P.timeout_ns) { rer = DEV_E_COMM; break; }
            }
            asm volatile("fence.acq_rel.sys;" ::: "memory");
            if (!rer) {
                rmin = ld_relaxed_sys(slot + 0);
                const u64 ce = ld_relaxed_sys(slot + 1);
                rT = (u32)ce; rer = (u32)(ce >> 32);
            }
        }
        const u64 xmin = warp_min_u64(rmin);
        const u32 xer = __reduce_or_sync(FULL, rer);
        const u32 cr = (lane < P.world && rmin == xmin) ? rT : 0u;
        Tg = __reduce_add_sync(FULL, cr);
        const u32 incl = warp_incl_scan(cr, lane);
        d.err = (int)xer;
        if (!xer && Tg > 0) {
            if (Tg > 1) { kk = tie_index(modtab, c0_lo, c0_hi, ties, Tg); ties += 1; }
            const u32 ge = __ballot_sync(FULL, lane < P.world && incl > kk && cr > 0);
            const int owner_rank = __ffs(ge) - 1;
            const u32 bef = owner_rank > 0 ? __shfl_sync(FULL, incl, owner_rank - 1) : 0u;
            mine = owner_rank == P.rank;
            kk -= bef;                            // this rank's local tie index if it owns
        }
        // sharded: every rank stamps each decision on its own clock (rank 0's series gives p50/p99)
        if (P.dec_ns != nullptr && cta == 0 && lane == 0) P.dec_ns[k] = (i64)globaltimer();
    } else if (!d.err && T > 1) {                 // TieBreaker.pick: tied[counter % len]; counter += 1
        kk = tie_index(modtab, c0_lo, c0_hi, ties, T);
        ties += 1;
    }
    if (!d.err && Tg == 0) d.err = 11;            // NoInstancesError
#ifdef RSIM_DIAG
    dt2 = clock64();
#endif
    if (!d.err && mine && single) {
        u32 pre = 0, kr = 0, bm = 0;
        int rb = -1;
#pragma unroll
        for (int r = 0; r < NRT; r++) {
            const u32 S = __popc(tb[r]);
            if (rb < 0 && kk < pre + S) { rb = r; kr = kk - pre; bm = tb[r]; }
            pre += S;
        }
        const int owner = rb * 32 + nth_set_bit_warp(bm, (int)kr, lane);
        if ((unsigned)(owner - cta * W) < (unsigned)W) { d.owner_warp = owner - cta * W; d.kk = 0; }   // (no division)
        d.oflat = owner; d.okk = 0;
    } else if (!d.err && mine) {
        // the round holding the kk-th tie, then the lane inside it
        u32 pre = 0, kr = 0, c = 0;
        int rb = -1;
#pragma unroll
        for (int r = 0; r < NRT; r++) {
            if (r < NR) {
                const u32 S = __reduce_add_sync(FULL, pc[r]);
                if (rb < 0 && kk < pre + S) { rb = r; kr = kk - pre; c = pc[r]; }
                pre += S;
            }
        }
        const u32 incl = warp_incl_scan(c, lane);
        const u32 ge = __ballot_sync(FULL, c > 0 && incl > kr && incl - c <= kr);
        const int L = __ffs(ge) - 1;
        const u32 okk = __shfl_sync(FULL, kr - (incl - c), L);
        const int owner = rb * 32 + L;
        if ((unsigned)(owner - cta * W) < (unsigned)W) { d.owner_warp = owner - cta * W; d.kk = (int)okk; }   // (no division)
        d.oflat = owner; d.okk = (int)okk;
    }
    d.pad = det_branch ? det_code : (bs_branch ? 1 : 0);   // the owner picks its tie among the chosen branch
#ifdef RSIM_DIAG
    dt3 = clock64();
    if (dg) { atomicAdd(P.ctr + 35, (u64)(dt1 - dt0)); atomicAdd(P.ctr + 36, (u64)(dt2 - dt1)); atomicAdd(P.ctr + 37, (u64)(dt3 - dt2)); }
#endif
    if (lane == 0) dec = d;
}

// The per-launch partial count fixes the rounds: instantiate the decide for 1, 2 or 4 rounds
// (api64: 16 x 4 partials = 2 rounds) instead of predicating 8.
__device__ __forceinline__ void decide_phase(const Params &P, const Part *part, int CW, int W, int cta, i64 k, int par,
                                             Dec &dec, u32 *modtab, u64 c0_lo, u64 c0_hi, u32 &ties, int lane,
                                             bool filter, const Part *det_branch = nullptr, int det_code = 0) {
    if (CW <= 32) decide_phase_n<1>(P, part, CW, W, cta, k, par, dec, modtab, c0_lo, c0_hi, ties, lane, filter, det_branch, det_code);
    else if (CW <= 64) decide_phase_n<2>(P, part, CW, W, cta, k, par, dec, modtab, c0_lo, c0_hi, ties, lane, filter, det_branch, det_code);
    else decide_phase_n<4>(P, part, CW, W, cta, k, par, dec, modtab, c0_lo, c0_hi, ties, lane, filter, det_branch, det_code);
}

__device__ __forceinline__ void bar_warps(int nthreads) {       // named barrier 1: the instance warps only
    asm volatile("bar.sync 1, %0;" :: "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------- replay
// Persistent launch over a cluster of C CTAs (C <= 16, one instance shard per
// CTA, engine state in shared memory, warps 0..W-1 own ipw instances each).
// Warp W of every CTA is the control warp: it stages requests into a
// shared-memory ring up to RSIM_SLOTS-1 decisions ahead and decides. Per
// decision k every instance warp
//   1. advances its instances through the engine steps starting before t_k,
//   2. takes each instance's hit blocks from the probe-ahead made during
//      decision k-1 when the instance's KV$ key set is unchanged since
//      (tabver), and probes the rest,
//   3. scores its instances and pushes one (min score, tie count) partial into
//      every CTA of the cluster with st.async (completing tx-bytes on the
//      receiver's mbarrier),
//   4. while the partials are in flight: advances instances that cannot win
//      k to t_{k+1}, then probes request k+1 against every instance
//      (probe-ahead; a commit only touches/pins, it never changes the key set),
// and the control warp of every CTA waits for the C*W partials, derives the
// same winner and releases the CTA through one barrier; the owning warp
// commits. No host round trip.
template <int MAXW, bool FILTER>      // FILTER: the two-branch partials of route_filter (policy 4)
__global__ void __launch_bounds__(32 * (MAXW + 1), 1)
replay_kernel(const __grid_constant__ Params P, i64 k0, i64 k1, i64 until, int mode, int target) {
    const int C = P.C, W = P.W, ipw = P.ipw, CW = P.C * P.W;
    // central mode: CTA C of the cluster is the decider (its control warp alone waits for the
    // partials, decides and st.async-broadcasts the decision to every instance CTA's release
    // mbarrier). Decide latency is sensitive to what else issues on its SM (measured: 4 warps
    // merely reading the landed partials next to it cost +4 % per decision), so it gets an SM of
    // its own, and each instance warp publishes one partial instead of C.
    const bool central = !FILTER && P.central != 0;
    const int CS = C + (central ? 1 : 0);                  // cluster size
    const int cta = (CS > 1) ? (int)cluster_ctarank() : 0;
    const bool decider = central && cta == C;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool control = warp == W;
    const int base = cta * P.per_cta;
    const int nloc = max(0, min(P.per_cta, P.N - base));
    Inst *st = (Inst *)smem;
    Part *part = (Part *)(st + P.per_cta);                 // [2 parity][2 branch][C*W], flat index cta*W + warp
    Part *part0 = part + 4 * CW;                           // [2 parity][C*W] round-0 partials (linear)
    ReqStage *rq = (ReqStage *)(part + 6 * CW);            // [RSIM_SLOTS] request ring (k % RSIM_SLOTS)
    Dec *dec = (Dec *)(rq + RSIM_SLOTS);                   // [2]
    u64 *mb = (u64 *)(dec + 2);                            // [2] partial-exchange mbarriers
    volatile i64 *ctl = (volatile i64 *)(mb + 2);          // [0] staged_upto
    u64 *dmb = mb + 4;                                     // [2] decision-release mbarriers (control -> CTA)
    u64 *mb0 = mb + 6;                                     // [2] round-0 mbarriers (linear, per-decision bs max)
    u32 *modtab = (u32 *)(mb + 8);                         // [RSIM_MODTAB] launch counter mod T
    WarpBuf *wbuf = (WarpBuf *)(modtab + RSIM_MODTAB);     // [W]
    WarpBuf &WB = wbuf[control ? 0 : warp];
    HistHead *hhc = (HistHead *)(wbuf + W);                // [per_cta] history heads (FILTER, staleness > 0)
    // hotspot detector: trace replays and route() decisions (an enqueue() API call does not involve it)
    const bool det = FILTER && P.dtid != nullptr && mode != MODE_ENQUEUE;
    DetCtl *dctl = (DetCtl *)(hhc + (P.stal > 0 ? P.per_cta : 0));
    Part *dpart = (Part *)(dctl + 1);                      // [2 parity][masked, least bs, products][C*W]
    unsigned char *ecnt = (unsigned char *)(dpart + 8 * CW);   // [2 parity][C*W][RSIM_DLMAX] listed holder counts
    const int BCd = 1 << P.dbclog2;
    DetView DV{P.dtr, P.dtkey, P.dglob, P.dbk + (size_t)cta * P.dTs * BCd * 3, P.dtot + (size_t)cta * BCd * 2, cta == 0};
    if (det && P.dsm) {                                    // tracks in shared memory (one copy per CTA)
        DV.tr = (DTrack *)(ecnt + 2 * CW * RSIM_DLMAX); DV.key = (const u64 *)(DV.tr + P.dT); DV.g = dctl->g;
    }
    const bool det_run = det && (mode == MODE_REPLAY || mode == MODE_ROUTE) && k0 < k1;

    {   // load this CTA's instance shard
        const u64 *src = (const u64 *)(P.inst + base);
        u64 *dst = (u64 *)st;
        const int words = nloc * (int)(sizeof(Inst) / 8);
        for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nloc; i += blockDim.x) {   // head caches start cold
        st[i].qcpos = -1;
        if (FILTER && P.stal > 0) { hhc[i].hidx = -1; hhc[i].ntidx = -1; }
    }
    const u64 c0_lo = P.tie[0], c0_hi = P.tie[1];          // TieBreaker counter at launch
    u32 ties = 0;                                          // ties resolved in this launch (control warp)
    const int l0 = warp * ipw;
    const int nmine = control ? 0 : max(0, min(ipw, nloc - l0));
    if (!control && lane == 0) { WB.c_bytes = 0; WB.c_steps = 0; WB.werr = 0; WB.fins = 0; WB.spk = -1; WB.fin.dnf = 0; WB.fin.npark = 0; WB.fin.tpn = 0; WB.fin.lnext = WB.fin.lend = 0; }
    if (threadIdx.x == 0) {
        // detector mode: every instance warp also arrives (release) after its plain shared-memory stores
        mbar_init(&mb[0], 1); mbar_init(&mb[1], 1); mbar_init(&dmb[0], 1); mbar_init(&dmb[1], 1);
        mbar_init(&mb0[0], 1); mbar_init(&mb0[1], 1);
        if (det) { mbar_init(&dctl->mbd[0], 1); mbar_init(&dctl->mbd[1], 1); }
        mbar_fence_init();
        ctl[0] = k0;
    }
    if (mode != MODE_DRAIN)
        for (int T = threadIdx.x; T < RSIM_MODTAB; T += blockDim.x) modtab[T] = 0xffffffffu;
    if (P.rsm_off) {                                       // running lists of this shard -> shared memory
        // (only the live prefix [0, r) of each list: the lists are kept compact)
        const int nw = blockDim.x >> 5;
        for (int i = warp; i < nloc; i += nw) {
            const ulonglong2 *src = reinterpret_cast<const ulonglong2 *>(P.rbuf + (size_t)(base + i) * P.max_batch);
            ulonglong2 *dst = reinterpret_cast<ulonglong2 *>(smem + P.rsm_off) + (size_t)i * P.max_batch * (sizeof(REnt) / 16);
            const int n16 = st[i].r * (int)(sizeof(REnt) / 16);
            for (int j = lane; j < n16; j += 32) dst[j] = src[j];
        }
    }
    if (det_run) {
        if (P.dsm) {                                        // detector state -> shared memory
            const int words = P.dT * (int)(sizeof(DTrack) / 8);
            for (int i = threadIdx.x; i < words; i += blockDim.x) ((i64 *)DV.tr)[i] = ((const i64 *)P.dtr)[i];
            for (int i = threadIdx.x; i < P.dT; i += blockDim.x) ((u64 *)DV.key)[i] = P.dtkey[i];
            for (int i = threadIdx.x; i < DG_N; i += blockDim.x) DV.g[i] = P.dglob[i];
        }
        __syncthreads();
        if (control) {                                      // verdict + list of k0
            det_prepare(P, DV, *dctl, P.arrival[k0], P.dtid[k0], P.dtw[P.dtid[k0]], lane);
            if (lane == 0) dctl->list_seq = (k0 << 8) | dctl->nl;
        }
    }
    __syncthreads();
    if (CS > 1) cluster_sync_all();

    // per-phase SM-cycle accounting of CTA 0 (ctr[8..15]): warp 0: staging wait, drain,
    // probe + score, publish + advance + probe-ahead, -, -, decision wait, commit;
    // control warp: exchange wait (4), decide (5)
    // (diagnostics builds only: -DRSIM_DIAG; they cost registers the production path needs)
#ifdef RSIM_DIAG
    const bool prof = P.ctr != nullptr && cta == 0 && (warp == 0 || control);
    u64 ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tc = clock64();
#define PHASE(i) do { if (prof) { const long long t2 = clock64(); ph[i] += (u64)(t2 - tc); tc = t2; } } while (0)
#define DIAG(x) x
#else
#define PHASE(i) do { } while (0)
#define DIAG(x)
#endif
    if (mode == MODE_DRAIN) {
        if (!control) drain_phase<FILTER, (RSIM_DECODE_RUNS >= 1)>(P, st, base, l0, nmine, until, 0u, lane, WB);
    } else if (central && decider) {
        if (control) {      // ---- the decider: partials of k -> decision -> every instance CTA
            u32 mb_phase = 0u;
            for (i64 k = k0; k < k1; k++) {
                const int par = (int)(k & 1);
                if (lane == 0) mbar_arrive_expect(&mb[par], (u32)(CW * 16));
                while (!mbar_try_wait(&mb[par], (mb_phase >> par) & 1u)) { }
                mb_phase ^= 1u << par;
#ifdef RSIM_DIAG
                u64 *tlc = (P.crit != nullptr && lane == 0 && k - k0 < P.crit_cap)
                               ? reinterpret_cast<u64 *>(P.crit + (size_t)P.crit_cap * CW * 8) + (size_t)(k - k0) * (CW + 4) + CW
                               : nullptr;
                if (tlc) tlc[0] = globaltimer();
#endif
                decide_phase(P, part, CW, W, 0, k, par, dec[par], modtab, c0_lo, c0_hi, ties, lane, false);
                __syncwarp();
#ifdef RSIM_DIAG
                if (tlc) tlc[1] = globaltimer();
#endif
                const Dec d = dec[par];   // (owner_warp, kk, err, pad) <- (flat owner, its tie index, err, branch)
                const u64 a = ((u64)(u32)d.okk << 32) | (u32)d.oflat;
                const u64 b = ((u64)(u32)d.pad << 32) | (u32)d.err;
                if (lane < C) st_async_16(&dec[par], &dmb[par], (u32)lane, a, b);
                if (d.err) break;
            }
        }
    } else if (central && control) {
        // ---- instance CTA's control warp: stage ahead; arm each decision's release mbarrier for
        //      the decider's 16-byte broadcast
        u32 dph_c = 0u;
        i64 staged = k0;
        auto stage_upto = [&](i64 lim) {
            lim = min(lim, k1);
            if (staged >= lim) return;
            while (staged < lim) { stage_request(P, rq[staged % RSIM_SLOTS], staged, mode, until, lane); staged++; }
            __threadfence_block();
            __syncwarp();
            if (lane == 0) ctl[0] = staged;
            __syncwarp();
        };
        stage_upto(k0 + RSIM_SLOTS - 1);
        for (i64 k = k0; k < k1; k++) {
            const int par = (int)(k & 1);
            if (lane == 0) mbar_arrive_expect(&dmb[par], 16u);
            while (!mbar_try_wait(&dmb[par], (dph_c >> par) & 1u)) { }
            dph_c ^= 1u << par;
            if (dec[par].err) break;
            // the decider had every warp's partial of k, so every warp committed k-1 and ran the
            // touch + pin of k-2: slots of decisions < k-1 are free
            stage_upto(k - 2 + RSIM_SLOTS);
        }
    } else if (control) {
        // ---- control warp: stage ahead, then per decision wait for the partials and decide
        u32 mb_phase = 0u;                                  // bit p: phase of mbarrier mb[p]
        u32 mbd_phase = 0u;                                 // bit p: phase of the detector barrier mbd[p]
        int det_hb = 0, det_code = 0;                       // decision k's chosen hit blocks, branch
        i64 det_pc = 0, det_nh = 0, det_psum = 0;           // its product; holders; holder-free product sum
        u64 det_pmin = ~0ULL;
        i64 staged = k0;
        auto stage_upto = [&](i64 lim) {
            lim = min(lim, k1);
            if (staged >= lim) return;
            while (staged < lim) { stage_request(P, rq[staged % RSIM_SLOTS], staged, mode, until, lane); staged++; }
            __threadfence_block();
            __syncwarp();
            if (lane == 0) ctl[0] = staged;
            __syncwarp();
        };
        stage_upto(k0 + RSIM_SLOTS - 1);
        for (i64 k = k0; k < k1; k++) {
            const int par = (int)(k & 1);
            DIAG(tc = clock64());
            const bool lin_dyn = FILTER && P.policy == 3 && !(P.bsn > 0);   // linear with the per-decision bs max
            if (lane == 0) {
                if (lin_dyn) mbar_arrive_expect(&mb0[par], (u32)(CW * 16));
                mbar_arrive_expect(&mb[par], (u32)(CW * (16 + (FILTER && P.policy == 4 ? 16 : 0) +
                                                         (det ? 48 + (FILTER && P.policy == 4 ? 16 : 0) : 0))));
                // the listed holder counts of every warp + the chosen instance's (hit, product) from its warp
                if (det) mbar_arrive_expect(&dctl->mbd[par], (u32)(CW * 16 * ((dctl->nl + 15) >> 4) + 16));
            }
            while (!mbar_try_wait(&mb[par], (mb_phase >> par) & 1u)) { }
            mb_phase ^= 1u << par;
            PHASE(4);
#ifdef RSIM_DIAG
            u64 *tlc = (P.crit != nullptr && cta == 0 && lane == 0 && k - k0 < P.crit_cap)
                           ? reinterpret_cast<u64 *>(P.crit + (size_t)P.crit_cap * CW * 8) + (size_t)(k - k0) * (CW + 4) + CW
                           : nullptr;
            if (tlc) tlc[0] = globaltimer();
#endif
            if (det) {     // verdict(k) -> argmin branch (policies.py:222-236), then observe(k) before the release
                const Part *dp = dpart + par * 4 * CW;
                i64 nh = 0, psum = 0;
                u64 pmin = ~0ULL;
                for (int i = lane; i < CW; i += 32) {
                    const ulonglong2 a = lds_v2u64(dp + i), c = lds_v2u64(dp + 2 * CW + i);
                    nh += (i64)(a.y >> 32); pmin = min(pmin, c.x); psum += (i64)c.y;
                }
                nh = warp_sum(nh); psum = warp_sum(psum); pmin = warp_min_u64(pmin);
                const int v = dctl->verdict;
                int code = v == 2 ? 3 : (v == 1 && nh < P.N ? 2 : 0);         // fail open when all hold
                if (FILTER && P.policy == 4 && code == 2) {
                    // route_filter over the kept (non-holder) candidates (policies.py:168-192, 229-236):
                    // their batch-size range picks least bs among them (code 4) or the hit branch (2)
                    u64 bmn = ~0ULL;
                    u32 bmx = 0;
                    for (int i = lane; i < CW; i += 32) {
                        const ulonglong2 q = lds_v2u64(dp + 3 * CW + i);
                        bmn = min(bmn, q.x); bmx = max(bmx, (u32)(q.y >> 32));
                    }
                    bmn = warp_min_u64(bmn);
                    bmx = __reduce_max_sync(FULL, bmx);
                    const i64 lo = bmn == ~0ULL ? 0 : (i64)__longlong_as_double((long long)bmn);
                    if ((i64)bmx - lo > P.range_thr) code = 4;
                }
                det_code = code;
                if (mode == MODE_ROUTE && P.scores != nullptr && cta == 0 && lane == 0) P.scores[5 * P.N] = (double)code;
                decide_phase(P, part, CW, W, cta, k, par, dec[par], modtab, c0_lo, c0_hi, ties, lane,
                             FILTER && P.policy == 4,
                             code == 2 ? dp : code == 3 ? dp + CW : code == 4 ? dp + 3 * CW : nullptr, code);
                __syncwarp();
                det_nh = nh; det_pmin = pmin; det_psum = psum;
            } else {
                decide_phase(P, part, CW, W, cta, k, par, dec[par], modtab, c0_lo, c0_hi, ties, lane, FILTER && P.policy == 4);
            }
            PHASE(5);
#ifdef RSIM_DIAG
            if (tlc) tlc[1] = globaltimer();
#endif
            __syncwarp();
            if (lane == 0) mbar_arrive(&dmb[par]);          // release decision k to the instance warps
            if (dec[par].err) break;
            if (det) {     // observe(k) and verdict / list of k+1 while the warps work on k+1
                DIAG(const long long tdw0 = clock64());
                while (!mbar_try_wait(&dctl->mbd[par], (mbd_phase >> par) & 1u)) { }   // listed holders counted
                mbd_phase ^= 1u << par;
                // the chosen instance's hit blocks and product, pushed by its warp after the release (a read of
                // the owner's buffers from here would race with that warp moving on to k+1)
                det_hb = (int)dctl->own[par][0];
                det_pc = (i64)dctl->own[par][1];
                const ReqStage &Rk = rq[k % RSIM_SLOTS];
                i64 ht = (i64)det_hb * P.bs; if (ht > Rk.in) ht = Rk.in;
                const int nl = dctl->nl;
                for (int j = lane; j < nl; j += 32) {       // listed holders, summed over the cluster's warps
                    u32 c = 0;
                    for (int w = 0; w < CW; w++) c += ecnt[((size_t)par * CW + w) * RSIM_DLMAX + j];
                    dctl->cnt[j] = c;
                }
                __syncwarp();
                if (P.ddbg != nullptr && lane == 0 && cta == 0) {
                    i64 *g = P.ddbg + (8 + P.N) * k;
                    g[0] = det_code; g[1] = det_nh; g[2] = (i64)det_pmin; g[3] = det_psum; g[4] = ht; g[5] = det_pc;
                    g[6] = det_hb >= Rk.dw; g[7] = nl;
                }
                DIAG(const long long tdw1 = clock64());
                if (det_pc >= 0)
                    det_observe(P, DV, *dctl, Rk.dtid, Rk.t, lane, ht, det_hb >= Rk.dw, det_pc, det_nh, det_pmin, det_psum,
                                dctl->cnt);
                DIAG(const long long tdw2 = clock64());
                if (k + 1 < k1) {
                    const ReqStage &Rn = rq[(k + 1) % RSIM_SLOTS];   // staged (slots up to k-2+RSIM_SLOTS)
                    det_prepare(P, DV, *dctl, Rn.t, Rn.dtid, Rn.dw, lane);
                    __threadfence_block();
                    if (lane == 0) *(volatile i64 *)&dctl->list_seq = ((k + 1) << 8) | dctl->nl;
                }
                DIAG(if (prof && lane == 0) { atomicAdd(P.ctr + 38, (u64)(tdw1 - tdw0)); atomicAdd(P.ctr + 39, (u64)(tdw2 - tdw1));
                                              atomicAdd(P.ctr + 40, (u64)(clock64() - tdw2)); atomicAdd(P.ctr + 41, (u64)(nl > 0)); });
            }
            // every warp published k, so it committed k-1 and ran the touch + pin of k-2
            // (which reads its request's staged keys): slots of decisions < k-1 are free
            stage_upto(k - 2 + RSIM_SLOTS);
        }
    } else if (!decider) {
        i64 staged_seen = k0;
        u32 dph = 0u;                                       // bit p: phase of decision-release mbarrier dmb[p]
        u32 d0ph = 0u;                                      // bit p: phase of round-0 mbarrier mb0[p]
        DIAG(long long t_rel = clock64());                  // release of this warp for decision k
        DIAG(bool was_owner = false);                       // this warp committed the previous decision
        for (i64 k = k0; k < k1; k++) {
            const int par = (int)(k & 1);
            DIAG(const u64 steps0 = WB.c_steps);
            DIAG(const int fins0 = WB.fins);
            DIAG(const int park0 = WB.fin.npark);
            if (staged_seen <= k) {                         // request k staged? normally long done
                while ((staged_seen = ctl[0]) <= k) { }
                __threadfence_block();
            }
            const ReqStage &R = rq[k % RSIM_SLOTS];
            PHASE(0);
            DIAG(const long long t_a = clock64());
            // ---- K4: advance my instances through steps starting before t; finisher cache work
            //      that cannot change this decision's probe beyond a closed-form update is parked
            Defer df;
            df.rkeys = R.keys; df.rB = R.B; df.hit = WB.sph; df.moved = 0u;
            df.valid = __ballot_sync(FULL, WB.spk == k && lane < nmine && st[l0 + lane].tabver == WB.spver[lane]);
            if (mode == MODE_REPLAY) drain_phase<FILTER>(P, st, base, l0, nmine, R.t, 0u, lane, WB, &df);
            PHASE(1);
            DIAG(const long long t_b = clock64());
            // ---- K2: hit blocks (probe-ahead where still valid) + score
            u32 skip = 0;
            if (WB.spk == k) {
                const bool ok = lane < nmine && st[l0 + lane].tabver == WB.spver[lane];
                if (ok) WB.hit[lane] = WB.sph[lane];
                skip = __ballot_sync(FULL, ok);
            }
            const u32 stale_slots = df.moved & skip;     // hits raised by a parked batch: no probe slots
            __syncwarp();
            if ((~skip & (nmine >= 32 ? FULL : ((1u << nmine) - 1u))) != 0) {   // (an out-of-line call: skip when idle)
                if (nmine >= 2 && R.B <= 128)
                    probe_hits_sparse(P, base, l0, nmine, R, mode, target, skip, lane, WB.hit);
                else
                    probe_hits(P, base, l0, nmine, R, mode, target, skip, lane, WB.hit, WB.slot[par]);
            }
            const u32 sparse_probe = (nmine >= 2 && R.B <= 128) ? ~skip : 0u;   // no probe slots for these
            const bool stale = FILTER && P.stal > 0;
            if (stale) {        // snapshot(now, staleness) of every candidate (indicators.py:36-65)
                const int gi = base + l0 + lane;
                if (lane < nmine && (mode != MODE_ENQUEUE || gi == target)) {
                    Inst &si = st[l0 + lane];
                    flush_view_hist(P, si, gi, R.t);
                    hist_snapshot(P, si, hhc[l0 + lane], gi, R.t - P.stal);
                }
                __syncwarp();
            }
            double bsn = P.bsn, bsn_kept = P.bsn;      // linear's normaliser over all / over the kept set
            if (FILTER && P.policy == 3 && !(P.bsn > 0)) {      // linear without a cap: bs_norm = max(max bs, 1) over ALL
                                                // instances (policies.py:250-255) -- one extra exchange round
                u32 lb = 0u, lbk = 0u;
                if (lane < nmine) {
                    const Inst *sp = st + l0 + lane;
                    lb = stale ? (u32)(hhc[l0 + lane].r + hhc[l0 + lane].q)
                               : sp->due <= R.t ? (u32)(sp->r + sp->q) : (u32)(sp->v_r + sp->v_q);
                    // detector: also the max over the non-holders of class(k), the set an exclusion keeps
                    if (!(det && WB.hit[lane] >= R.dw)) lbk = lb;
                }
                lb = __reduce_max_sync(FULL, lb);
                lbk = __reduce_max_sync(FULL, lbk);
                if (lane < C) st_async_16(part0 + par * CW + cta * W + warp, &mb0[par], (u32)lane, (u64)lb, (u64)lbk);
                while (!mbar_try_wait(&mb0[par], (d0ph >> par) & 1u)) { }
                d0ph ^= 1u << par;
                u32 gm = 0u, gmk = 0u;
                for (int i = lane; i < CW; i += 32) {
                    const ulonglong2 q = lds_v2u64(part0 + par * CW + i);
                    gm = max(gm, (u32)q.x); gmk = max(gmk, (u32)q.y);
                }
                gm = __reduce_max_sync(FULL, gm);
                gmk = __reduce_max_sync(FULL, gmk);
                if (P.world > 1) {      // the max is over ALL instances: one more mailbox round
                    const u64 seq = (P.epoch << 40) | (u64)(k + 1);   // (words 3, 4, 7 of the slot)
                    if (cta == 0 && warp == 0 && lane < P.world) {
                        u64 *slot = P.peer[lane] + (size_t)((par * 8 + P.rank) * RSIM_MBOX_W);
                        st_relaxed_sys(slot + 3, (u64)gm);
                        st_relaxed_sys(slot + 4, (u64)gmk);
                        st_release_sys(slot + 7, seq);
                    }
                    u32 rg = 0u, rgk = 0u, rer = 0u;
                    if (lane < P.world) {
                        const u64 *slot = P.mbox + (size_t)((par * 8 + lane) * RSIM_MBOX_W);
                        const u64 tt = globaltimer();
                        while (ld_relaxed_sys(slot + 7) != seq) {
                            if ((i64)(globaltimer() - tt) > P.timeout_ns) { rer = DEV_E_COMM; break; }
                        }
                        asm volatile("fence.acq_rel.sys;" ::: "memory");
                        if (!rer) { rg = (u32)ld_relaxed_sys(slot + 3); rgk = (u32)ld_relaxed_sys(slot + 4); }
                    }
                    gm = __reduce_max_sync(FULL, rg);
                    gmk = __reduce_max_sync(FULL, rgk);
                    if (__reduce_or_sync(FULL, rer) && lane == 0) WB.werr = DEV_E_COMM;
                }
                bsn = (double)(gm > 1u ? gm : 1u);
                bsn_kept = (double)(gmk > 1u ? gmk : 1u);
            }
            u64 bits_bs;
            const u64 mybits = score_phase(P, st, base, l0, nmine, R, mode, target, lane, WB, bits_bs,
                                           FILTER && P.policy == 4, bsn, stale, hhc, det,
                                           FILTER && P.policy == 5 ? P.simj + ((size_t)(cta * W + warp) << P.qlog2)
                                                                   : nullptr);
            PHASE(2);
            DIAG(const long long t_c = clock64());
            if (cta == 0 && warp == 0 && lane == 0) WB.c_bytes += 8ULL * (u64)R.B;   // request chain keys, read once
            const u32 whi = __reduce_min_sync(FULL, (u32)(mybits >> 32));
            const u64 wmin = ((u64)whi << 32) | __reduce_min_sync(FULL, (u32)(mybits >> 32) == whi ? (u32)mybits : ~0u);
            const u32 tmask = __ballot_sync(FULL, lane < nmine && mybits == wmin && wmin != ~0ULL);
            u64 wmin_bs = ~0ULL;
            u32 tmask_bs = 0u;
            if (FILTER && P.policy == 4) {               // filter: both branches, decided globally
                const u32 bhi = __reduce_min_sync(FULL, (u32)(bits_bs >> 32));
                wmin_bs = ((u64)bhi << 32) | __reduce_min_sync(FULL, (u32)(bits_bs >> 32) == bhi ? (u32)bits_bs : ~0u);
                tmask_bs = __ballot_sync(FULL, lane < nmine && bits_bs == wmin_bs && wmin_bs != ~0ULL);
            }
            u32 det_keep = 0u;
            int det_nl = 0;          // |list| of decision k (the control warp rewrites it for k+1 once
                                     // every warp has sent k's counts)
            if (det) {     // detector partials (rsim_detector.cuh): plain stores + a release arrive (C == 1)
                const bool cand = lane < nmine;
                const bool held = cand && WB.hit[lane] >= R.dw;          // holders of class(k)
                u64 kb = mybits;                          // the kept-set score (uncapped linear renormalises)
                if (FILTER && P.policy == 3 && !(P.bsn > 0) && cand && !held) {
                    kb = (u64)__double_as_longlong(score_of(P, WB.bsv[lane], 0, 0, 0, WB.hit[lane], R.in, bsn_kept));
                    if (mode == MODE_ROUTE && P.scores != nullptr) P.scores[4 * P.N + base + l0 + lane] = __longlong_as_double((long long)kb);
                }
                const u64 bx = (cand && !held) ? kb : ~0ULL;
                const u64 bl = cand ? (u64)__double_as_longlong((double)WB.bsv[lane]) : ~0ULL;
                const u64 pn = (cand && !held) ? (u64)WB.prod[lane] : ~0ULL;
                const i64 ps = warp_sum((cand && !held) ? WB.prod[lane] : 0LL);
                const u64 mx = warp_min_u64(bx), ml = warp_min_u64(bl), mp = warp_min_u64(pn);
                const u32 tx = __ballot_sync(FULL, cand && bx == mx && mx != ~0ULL);
                const u32 tl = __ballot_sync(FULL, cand && bl == ml && ml != ~0ULL);
                const u32 nhw = (u32)__popc(__ballot_sync(FULL, held));
                u32 txb = 0u;
                if (FILTER && P.policy == 4) {           // filter's bs branch among the non-holders
                    const u64 bb = (cand && !held) ? bits_bs : ~0ULL;
                    const u64 mb_ = warp_min_u64(bb);
                    txb = __ballot_sync(FULL, cand && !held && bb == mb_ && mb_ != ~0ULL);
                    const u32 bmx = __reduce_max_sync(FULL, (cand && !held) ? (u32)WB.bsv[lane] : 0u);
                    Part *dq = dpart + par * 4 * CW + 3 * CW + cta * W + warp;
                    if (lane < C) st_async_16(dq, &mb[par], (u32)lane, mb_, ((u64)bmx << 32) | (u32)__popc(txb));
                }
                det_keep = tx | tl | txb;
                if (P.ddbg != nullptr && cand) P.ddbg[(8 + P.N) * k + 8 + base + l0 + lane] = held ? -2 : WB.prod[lane];
                if (lane == 0) { WB.tm[0] = tmask; WB.tm[1] = tmask_bs; WB.tm[2] = tx; WB.tm[3] = tl; WB.tm[4] = txb; }
                __syncwarp();
                Part *dp = dpart + par * 4 * CW + cta * W + warp;
                if (lane < C) {
                    st_async_16(dp, &mb[par], (u32)lane, mx, ((u64)nhw << 32) | (u32)__popc(tx));
                    st_async_16(dp + CW, &mb[par], (u32)lane, ml, (u64)(u32)__popc(tl));
                    st_async_16(dp + 2 * CW, &mb[par], (u32)lane, mp, (u64)ps);
                }
            }
            {   // publish this warp's partial(s) to every CTA of the cluster
                const u64 w1 = ((u64)(u32)WB.werr << 32) | (u32)__popc(tmask);
                Part *dst = part + par * 2 * CW + cta * W + warp;
                if (central) { if (lane == 0) st_async_16(dst, &mb[par], (u32)C, wmin, w1); }   // the decider
                else if (lane < C) st_async_16(dst, &mb[par], (u32)lane, wmin, w1);
                if (FILTER && P.policy == 4) {           // second partial: (min bs, ties | max bs << 32)
                    const Inst &sv = st[l0 + lane];
                    const u32 bsmax = __reduce_max_sync(FULL, lane < nmine ? (u32)(stale ? hhc[l0 + lane].r + hhc[l0 + lane].q : sv.v_r + sv.v_q) : 0u);
                    const u64 w2 = ((u64)bsmax << 32) | (u32)__popc(tmask_bs);
                    if (lane < C) st_async_16(dst + CW, &mb[par], (u32)lane, wmin_bs, w2);
                }
            }
#ifdef RSIM_DIAG
            if (P.crit != nullptr && lane == 0 && k - k0 < P.crit_cap) {   // diagnostics: where this warp's latency went
                const long long t_d = clock64();
                auto q16 = [](long long c) { c >>= 4; return (unsigned short)(c > 65535 ? 65535 : (c < 0 ? 0 : c)); };
                unsigned short *rec = P.crit + ((size_t)(k - k0) * CW + cta * W + warp) * 8;
                rec[0] = q16(t_d - t_rel); rec[1] = q16(t_b - t_a); rec[2] = q16(t_c - t_b); rec[3] = q16(t_a - t_rel);
                rec[4] = (unsigned short)min((u64)65535, WB.c_steps - steps0); rec[5] = (unsigned short)(WB.fins - fins0);
                rec[6] = (unsigned short)(was_owner ? 1 : 0); rec[7] = (unsigned short)(WB.fin.npark - park0);
                u64 *tl = reinterpret_cast<u64 *>(P.crit + (size_t)P.crit_cap * CW * 8);
                tl[(size_t)(k - k0) * (CW + 4) + cta * W + warp] = globaltimer();
            }
#endif
            apply_deferred(P, WB.fin, lane, &WB.werr);      // parked finisher cache work (before any commit)
            flush_touch_pin(P, WB.fin, lane, &WB.werr);     // the previous commit's touch + pin
            if (det) {     // the control warp lists decision k's tracks after observe(k-1)
                i64 lw;
                while (((lw = *(volatile i64 *)&dctl->list_seq) >> 8) < k) { }
                __threadfence_block();
                // past k already: k's list was empty (a listed decision waits for every warp's counts)
                det_nl = (lw >> 8) == k ? (int)(lw & 0xff) : 0;
            }
            if (det && det_nl > 0) {     // holders of the listed tracks on the tables as of t_k (before any advance)
                const DetCtl &dc = *dctl;
                const int nl = det_nl, nch = (nl + 15) >> 4;
                for (int j = 0; j < nch * 16; j++) {
                    const bool hd = j < nl && lane < nmine && det_holds(P, dc.lst[j], base + l0 + lane);
                    const u32 c = (u32)__popc(__ballot_sync(FULL, hd));
                    if (lane == 0) WB.ecs[j] = (unsigned char)c;
                }
                __syncwarp();
                for (int q = 0; q < nch; q++) {
                    const ulonglong2 v = lds_v2u64(WB.ecs + 16 * q);
                    if (lane < C) st_async_16(ecnt + ((size_t)par * CW + cta * W + warp) * RSIM_DLMAX + 16 * q,
                                              &dctl->mbd[par], (u32)lane, v.x, v.y);
                }
            }
            if (mode == MODE_REPLAY && k + 1 < k1) {
                if (staged_seen <= k + 1) { staged_seen = ctl[0]; __threadfence_block(); }
                if (staged_seen > k + 1) {
                    const ReqStage &R1 = rq[(k + 1) % RSIM_SLOTS];
                    // instances that cannot win this decision advance to the next arrival meanwhile
                    const u32 adv = __ballot_sync(FULL, lane < nmine && mybits != wmin &&
                                                            (!(FILTER && P.policy == 4) || bits_bs != wmin_bs)) &
                                    ~det_keep;      // detector: the other argmin branches' candidates stay
                    DIAG(const long long t_s0 = clock64());
                    if (adv) drain_phase<FILTER, (RSIM_DECODE_RUNS >= 1)>(P, st, base, l0, nmine, R1.t, ~adv, lane, WB);
                    DIAG(const long long t_s1 = clock64());
                    // probe-ahead of request k+1 (valid while the instance's tabver holds)
                    if (nmine >= 2 && R1.B <= 128) {   // (one instance: the dense probe's single round trip wins)
                        probe_hits_sparse(P, base, l0, nmine, R1, mode, target, 0u, lane, WB.sph);
                    } else {
#ifdef RSIM_DIAG
                        probe_hits(P, base, l0, nmine, R1, mode, target, 0u, lane, WB.sph, WB.slot[par ^ 1], prof && warp == 0);
#else
                        probe_hits(P, base, l0, nmine, R1, mode, target, 0u, lane, WB.sph, WB.slot[par ^ 1]);
#endif
                    }
                    DIAG(if (prof && lane == 0) { atomicAdd(P.ctr + 30, (u64)(t_s1 - t_s0)); atomicAdd(P.ctr + 31, (u64)(clock64() - t_s1)); });
                    if (lane < nmine) WB.spver[lane] = st[l0 + lane].tabver;
                    if (lane == 0) WB.spk = k + 1;
                    __syncwarp();
                }
            }
            PHASE(3);
            while (!mbar_try_wait(&dmb[par], (dph >> par) & 1u)) { }   // decision k released by the control warp
            dph ^= 1u << par;
            PHASE(6);
#ifdef RSIM_DIAG
            if (P.crit != nullptr && cta == 0 && warp == 0 && lane == 0 && k - k0 < P.crit_cap)
                reinterpret_cast<u64 *>(P.crit + (size_t)P.crit_cap * CW * 8)[(size_t)(k - k0) * (CW + 4) + CW + 2] = globaltimer();
#endif
            DIAG(t_rel = clock64());
            Dec d = dec[par];
            if (central) {                                  // the broadcast names the owner by flat warp index
                const int ow = d.owner_warp - cta * W;
                d.owner_warp = (unsigned)ow < (unsigned)W ? ow : -1;
            }
            if (d.err) {
                if (lane == 0 && WB.werr == 0) WB.werr = d.err;
                break;
            }
            DIAG(was_owner = warp == d.owner_warp);
            if (warp == d.owner_warp) {
                const int s = nth_set_bit_warp(d.pad == 0 ? tmask : d.pad == 1 ? tmask_bs : WB.tm[d.pad], d.kk, lane);   // d.pad: the branch
                const int h = WB.hit[s];
                const int gch = P.gbase + base + l0 + s;
                const bool dup = mode == MODE_ROUTE && P.dupmask != nullptr && ((P.dupmask[gch >> 5] >> (gch & 31)) & 1u);
                // (hit, product) of the chosen instance to every CTA's observe(k); a duplicate request
                // is refused by enqueue before observe runs (cluster.py:140-142): product -1
                if (det && lane < C)
                    st_async_16(&dctl->own[par][0], &dctl->mbd[par], (u32)lane, (u64)(u32)h, dup ? ~0ULL : (u64)WB.prod[s]);
                int werr = 0;
                flush_touch_pin(P, WB.fin, lane, &WB.werr);      // (normally already run after the publish)
                if (dup) {
                    if (lane == 0) WB.werr = DEV_E_DUPLICATE;          // chosen (the counter moved), never enqueued
                } else
                commit(P, st + l0 + s, base + l0 + s, k, h, R.t, R.keys,
                       (s < 2 && nmine < 2 && !(((stale_slots | sparse_probe) >> s) & 1u)) ? WB.slot[par][s] : nullptr,
                       R.a, R.B, R.in, R.out, R.oa, lane, werr, WB.fin, FILTER && P.stal > 0);
                if (lane == 0 && werr) WB.werr = werr;
                if (P.dec_ns != nullptr && lane == 0 && P.world == 1) P.dec_ns[k] = (i64)globaltimer();
            }
            PHASE(7);
        }
    }
#undef PHASE
    if (!control && mode != MODE_DRAIN) flush_touch_pin(P, WB.fin, lane, &WB.werr);
    if (!control) close_log(P, WB.fin, lane);
#ifdef RSIM_DIAG
    if (prof && lane == 0)
        for (int i = 0; i < 8; i++) if (ph[i]) atomicAdd(P.ctr + 8 + i, ph[i]);
#endif
#undef DIAG
    // write back
    __syncthreads();
    if (det_run && P.dsm && cta == 0) {
        const int words = P.dT * (int)(sizeof(DTrack) / 8);
        for (int i = threadIdx.x; i < words; i += blockDim.x) ((i64 *)P.dtr)[i] = ((const i64 *)DV.tr)[i];
        for (int i = threadIdx.x; i < DG_N; i += blockDim.x) P.dglob[i] = DV.g[i];
    }
    {
        u64 *dst = (u64 *)(P.inst + base);
        const u64 *src = (const u64 *)st;
        const int words = nloc * (int)(sizeof(Inst) / 8);
        for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
    }
    if (P.rsm_off) {
        const int nw = blockDim.x >> 5;
        for (int i = warp; i < nloc; i += nw) {
            ulonglong2 *dst = reinterpret_cast<ulonglong2 *>(P.rbuf + (size_t)(base + i) * P.max_batch);
            const ulonglong2 *src = reinterpret_cast<const ulonglong2 *>(smem + P.rsm_off) + (size_t)i * P.max_batch * (sizeof(REnt) / 16);
            const int n16 = st[i].r * (int)(sizeof(REnt) / 16);
            for (int j = lane; j < n16; j += 32) dst[j] = src[j];
        }
    }
    if (!control && lane == 0) {
        if (WB.werr) atomicCAS(P.err, 0, WB.werr);
        if (P.ctr != nullptr) {
            if (WB.c_bytes) atomicAdd(P.ctr + 0, WB.c_bytes);
            if (WB.c_steps) atomicAdd(P.ctr + 1, WB.c_steps);
        }
    }
    if ((central ? decider : cta == 0) && control && lane == 0 && mode != MODE_DRAIN) {
        const u64 lo = c0_lo + ties;
        P.tie[0] = lo;
        P.tie[1] = c0_hi + (lo < c0_lo);
    }
    if (CS > 1) cluster_sync_all();
}

// ---------------------------------------------------------------- probe batch
// What-if probe (SURVEY 8d tertiary): M requests x all instances against the frozen state,
// no commits -- the bandwidth-bound form of the probe. One THREAD per (request, instance) pair
// walks the request's chain from depth 0 exactly as match_keys does (kvcache.py:65-74): one
// table lookup per depth, stop at the first miss, so a pair costs the reference's own
// min(h+1, B) lookups. Throughput comes from the number of independent walks in flight (every
// resident thread has its own), not from splitting one walk over a warp -- the warp-split
// probes of the replay kernel spend 8-16 lookups per pair to cut latency, which a batch does
// not need. The next D - 1 depths' pairs are in flight while one is evaluated (the up to D - 1
// lookups past the first miss are the only work beyond the reference's).
// Lanes of a warp take consecutive instances of one request: the request's chain keys are
// shared loads (L1 broadcast), the table lines are 32 independent sectors.
template <int D>      // lookups in flight per thread (D - 1 depths ahead of the one evaluated)
__global__ void __launch_bounds__(256)
probe_scan_kernel(const __grid_constant__ Params P, i64 r0, i64 nreq, int *out) {
    const i64 total = nreq * (i64)P.N;
    const i64 stride = (i64)gridDim.x * blockDim.x;
    const bool narrow = total <= 0xffffffffLL;               // 32-bit pair -> (request, instance)
    for (i64 p = (i64)blockIdx.x * blockDim.x + threadIdx.x; p < total; p += stride) {
        const i64 rr = narrow ? (i64)((u32)p / (u32)P.N) : p / P.N;
        const int gi = (int)(p - rr * P.N);
        const i64 a = __ldg(P.blk_off + r0 + rr);
        const int B = (int)(__ldg(P.blk_off + r0 + rr + 1) - a);
        const u64 *keys = P.ckeys + a;
        const Table T = table_of(P, gi);
        u64 kq[D];
        u32 hq[D];
        ulonglong2 pq[D];
#pragma unroll
        for (int j = 0; j < D; j++) {
            kq[j] = j < B ? __ldg(keys + j) : 0ULL;
            hq[j] = tab_home(kq[j], T.slog2);
            pq[j] = j < B ? ld_pair(T, hq[j]) : make_ulonglong2(0ULL, 0ULL);
        }
        int h = 0;
        bool go = true;
        while (go) {
#pragma unroll
            for (int j = 0; j < D; j++) {                     // slot j holds depth h (h % D == j)
                bool f, c;
                eval_first(T, pq[j], hq[j], kq[j], f, c);
                if (c) {
                    int stt;
                    probe_rest(T, ((hq[j] | 1u) + 1u) & T.mask, kq[j], stt);
                    f = stt == 0;
                }
                if (!f || ++h == B) { go = false; break; }
                const int d = h + D - 1;                      // refill: D - 1 depths ahead
                if (d < B) {
                    kq[j] = __ldg(keys + d);
                    hq[j] = tab_home(kq[j], T.slog2);
                    pq[j] = ld_pair(T, hq[j]);
                }
            }
        }
        out[p] = h;
    }
}

// ---------------------------------------------------------------- cache ops (API)
// op 0: insert_keys(keys, now) -> evicted ; op 1: match_keys(keys) -> hit.
// keys = P.arena + a0 (API keys persist in the arena so eviction runs can name them).
__global__ void cache_op_kernel(Params P, int gi, int op, i64 a0, int n, i64 now, i64 *result) {
    const int lane = threadIdx.x & 31;
    Table T = table_of(P, gi);
    const u64 *keys = P.arena + a0;
    int werr = 0;
    if (op == 1) {
        int h = warp_probe(T, keys, n, lane);
        if (lane == 0) result[0] = h;
        return;
    }
    Inst s = P.inst[gi];
    s.tabver += 1;
    if (n > 0) {
        Run r; r.T = now; r.a = a0; r.oa = 0; r.B = n; r.dhi = n; r.kind = 1; r.pad = 0;
        run_add(P, s, gi, r, lane, werr);
    }
    s.occ += warp_unpin_insert(T, keys, n, keys, n, 0, now, lane, werr);
    const i64 before_evict = s.occ;
    if (s.occ > P.max_occ) werr = DEV_E_TABLE_FULL;
    evict_to_capacity(P, T, s, gi, lane, werr);
    __syncwarp();
    if (lane == 0) {
        P.inst[gi] = s;
        result[0] = before_evict - s.occ;
        if (werr) atomicCAS(P.err, 0, werr);
    }
}
