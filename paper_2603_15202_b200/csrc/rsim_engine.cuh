// rsim_engine.cuh -- one instance's engine step, executed by its owning warp.
//
// Restates InstanceSim.form_batch + execute_batch (reference engine.py:291-355)
// with the cost model of engine.py:81-96, on the instance's state held in
// shared memory. FIFO chunked-prefill allocation is a warp prefix sum over
// the queue head; decode bookkeeping is O(1) per step because each running
// request's finish step is known when it joins (finish = join + out - 1), so
// the running list is only scanned on steps where something finishes.
#pragma once
#include "rsim_lru.cuh"

// Python round() of the double expression, evaluated in the reference's
// operation order with explicit round-to-nearest ops (no FMA contraction).
__device__ __forceinline__ i64 prefill_cost_us(const Params &P, i64 tok) {
    if (tok <= 0) return 0;
    double x = __dmul_rn(__dadd_rn(P.pb, __dmul_rn(P.pt, __ll2double_rn(tok))), 1000.0);
    return __double2ll_rn(x);
}
__device__ __forceinline__ i64 decode_cost_us(const Params &P, i64 n, i64 ctx) {
    if (n <= 0) return 0;
    double x = __dadd_rn(__dadd_rn(P.db, __dmul_rn(P.ds, __ll2double_rn(n))),
                         __dmul_rn(P.dcc, __ll2double_rn(ctx)));
    return __double2ll_rn(__dmul_rn(x, 1000.0));
}

// ---------------- simulate policy: TTFT replay (engine.py:419-460) ----------------
// estimate_first_token_us over sched_clone (engine.py:376-391) of instance gi, warp-wide:
// the live queue (ring, pending as of now) and running list replayed forward step by step
// under the policy's cost model (Policy.sim_cost_model, policies.py:206-211) with the
// candidate (pending max(cand, 1), in 0, out 1) appended FIFO-last; returns the absolute
// time of the candidate's first token (-1 past _REPLAY_STEP_CAP). Nothing is written back.
// Decode set at replay step s (running <= max_batch, so decode == running): a running
// entry with finish step v decodes in steps 0 .. v - step_idx with context
// in + out - (v - step_idx + 1) + s; a request popped at step j with out > 1 joins for
// steps j+1 .. j+out-1 with context in + 1 + (s - j - 1) (kept in the warp's scratch jb).
__device__ __forceinline__ i64 sim_prefill_us(const Params &P, i64 tok) {
    if (tok <= 0) return 0;
    return __double2ll_rn(__dmul_rn(__dadd_rn(P.spb, __dmul_rn(P.spt, __ll2double_rn(tok))), 1000.0));
}
__device__ __forceinline__ i64 sim_decode_us(const Params &P, i64 n, i64 ctx) {
    if (n <= 0) return 0;
    const double x = __dadd_rn(__dadd_rn(P.sdb, __dmul_rn(P.sds, __ll2double_rn(n))), __dmul_rn(P.sdc, __ll2double_rn(ctx)));
    return __double2ll_rn(__dmul_rn(x, 1000.0));
}
__device__ __noinline__ i64 sim_first_token(const Params &P, const Inst *sp, int gi, i64 now, i64 cand, int lane,
                                            int4 *jb) {
    const i64 S = sp->step_idx;
    const int nr = sp->r, q = sp->q, qh0 = sp->q_head;
    const QEnt *qb = P.qbuf + ((size_t)gi << P.qlog2);
    const REnt *rb = rlist(P, gi);
    const u32 qmask = (1u << P.qlog2) - 1u;
    const i64 pc = cand > 1 ? cand : 1;
    i64 t = now > sp->busy_until ? now : sp->busy_until;
    int qpos = 0;                                   // first queue entry not yet popped (q = the candidate)
    i64 hrem = q > 0 ? qb[qh0 & qmask].v : pc;      // its pending
    int nj = 0;                                     // joined requests in jb
    for (int s = 0; s < 10000000; s++) {            // _REPLAY_STEP_CAP
        i64 n = 0, ctx = 0;
        for (int i = lane; i < nr; i += 32) {
            const i64 er = rb[i].v - S;             // last replay step this entry decodes in
            if (er >= s) { n++; ctx += rb[i].in + (i64)rb[i].out - (er + 1) + s; }
        }
        for (int i = lane; i < nj; i += 32) {
            const int4 j = jb[i];
            if (j.x <= s && s <= j.y) { n++; ctx += (i64)j.z + (s - j.x); }
        }
        n = warp_sum(n); ctx = warp_sum(ctx);
        const i64 budget0 = P.chunk - n > 0 ? P.chunk - n : 0;   // engine.py:436-440
        const i64 slots = P.max_batch - n;
        // _plan_allocations over entries qpos.. (engine.py:174-184): entry j is allocated iff
        // j - qpos < slots and the budget left before it is positive; allocations form a prefix,
        // all popped (take == pending) except possibly the last
        i64 ptok = 0, spent = 0, nrem = -1;
        int npop = 0;
        bool cand_done = false;
        for (int w0 = qpos; w0 <= q; w0 += 32) {
            const int j = w0 + lane;
            const bool ex = j <= q;
            i64 p = 0;
            int jin = 0, jout = 1;
            if (ex) {
                if (j == q) p = pc;
                else {
                    const QEnt &e = qb[(qh0 + j) & qmask];
                    p = j == qpos ? hrem : e.v; jin = (int)e.in; jout = e.out;
                }
                if (j == qpos) p = hrem;
            }
            const i64 incl = warp_incl_scan(p, lane);
            const i64 before = budget0 - (spent + incl - p);
            const bool alloc = ex && (i64)(j - qpos) < slots && before > 0;
            const i64 take = alloc ? (before < p ? before : p) : 0;
            const bool popped = alloc && take == p;
            const u32 am = __ballot_sync(FULL, alloc), pm = __ballot_sync(FULL, popped);
            ptok += warp_sum(take);
            spent += __shfl_sync(FULL, incl, 31);
            if (__ballot_sync(FULL, popped && j == q)) cand_done = true;
            // requests that finish prefill join the decode set from the next step (engine.py:452-453)
            const bool joins = popped && j < q && jout > 1;
            const u32 jm = __ballot_sync(FULL, joins);
            if (joins) jb[nj + __popc(jm & lanemask_lt())] = make_int4(s + 1, s + jout - 1, jin + 1, 0);
            nj += __popc(jm);
            npop += __popc(pm);
            const u32 part = am & ~pm;                               // the partially allocated entry
            if (part) nrem = __shfl_sync(FULL, p - take, __ffs(part) - 1);
            if (am != FULL) break;                                   // the allocated prefix ended here
        }
        const i64 end = t + sim_prefill_us(P, ptok) + sim_decode_us(P, n, ctx);
        if (cand_done) return end;
        qpos += npop;
        if (nrem >= 0) hrem = nrem;
        else if (npop > 0) hrem = qpos == q ? pc : qb[(qh0 + qpos) & qmask].v;
        t = end;
        __syncwarp();
    }
    return -1;
}

__device__ __forceinline__ void flush_view(Inst &s, i64 now) {   // engine.py:240-246
    if (s.due <= now) {
        s.v_r = s.r; s.v_q = s.q; s.v_pend = s.pend; s.v_total = s.total; s.v_dc = s.dcs;
        s.due = RSIM_NONE;
    }
}
// the same, recording the flushed view in the history (engine.py:245; staleness > 0)
__device__ __forceinline__ void flush_view_hist(const Params &P, Inst &s, int gi, i64 now) {
    if (s.due <= now) {
        s.v_r = s.r; s.v_q = s.q; s.v_pend = s.pend; s.v_total = s.total; s.v_dc = s.dcs;
        hist_append(P, s, gi, s.due, now);
        s.due = RSIM_NONE;
    }
}

// _finish (engine.py:357-372) for one request: unpin the admission hit, insert
// the full prefix+output chain stamped with the step end, evict to capacity.
__device__ __forceinline__ void evict_to_capacity(const Params &P, const Table &T, Inst &s, int gi, int lane,
                                                  int &werr) {
    if (P.cap >= 0 && s.occ > P.cap && !werr)
        if (!evict_runs(P, T, s, gi, s.occ, lane, werr)) warp_evict(T, P.cap, s.occ, lane, werr);
}

__device__ void finish_one(const Params &P, int gi, Inst &s, i64 a, int B, i64 oa, int L, int hb, i64 end, int lane,
                           int &werr) {
    Table T = table_of(P, gi);
    Run r; r.T = end; r.a = a; r.oa = oa; r.B = B; r.dhi = L; r.kind = 0; r.pad = 0;
    run_add(P, s, gi, r, lane, werr);
#ifdef RSIM_STEP_PROFILE
    const long long c0 = clock64();
#endif
    s.occ += warp_unpin_insert(T, P.ckeys + a, B, P.okeys + oa, L, hb, end, lane, werr);
    if (s.occ > P.max_occ) werr = DEV_E_TABLE_FULL;
#ifdef RSIM_STEP_PROFILE
    const long long c1 = clock64();
#endif
    evict_to_capacity(P, T, s, gi, lane, werr);
#ifdef RSIM_STEP_PROFILE
    if (P.ctr != nullptr && lane == 0) { atomicAdd(P.ctr + 42, (u64)(c1 - c0)); atomicAdd(P.ctr + 43, (u64)(clock64() - c1)); }
#endif
}

// Process the finishers collected in F, in collection order (= the reference's:
// queue-pop finishes, then decode finishes in running order). When no eviction
// can happen before the last insert, all chains go in one batched pass.
__device__ void flush_finishers(const Params &P, int gi, Inst &s, FinBuf &F, int nf, i64 end, int lane, int &werr) {
    if (nf == 0 || werr) return;
    const long long c0 = clock64();
    s.tabver += 1;                                                 // invalidates probes made before this step
    __syncwarp();
    if (P.cap < 0 || s.occ + F.pre[nf] <= P.cap) {
        Table T = table_of(P, gi);
        for (int f = 0; f < nf; f++) {
            Run r; r.T = end; r.a = F.a[f]; r.oa = F.oa[f]; r.B = F.B[f]; r.dhi = F.L[f]; r.kind = 0; r.pad = 0;
            run_add(P, s, gi, r, lane, werr);
        }
        s.occ += warp_finish_many(T, P.ckeys, P.okeys, F, nf, end, lane, werr);
        if (s.occ > P.max_occ) werr = DEV_E_TABLE_FULL;
    } else {
        for (int f = 0; f < nf && !werr; f++)
            finish_one(P, gi, s, F.a[f], F.B[f], F.oa[f], F.L[f], F.hb[f], end, lane, werr);
    }
    __syncwarp();
    if (P.ctr != nullptr && lane == 0) { atomicAdd(P.ctr + 3, (u64)(clock64() - c0)); atomicAdd(P.ctr + 6, (u64)1); }
}

// The step log (record_steps): each warp reserves RSIM_LOG_CHUNK records at a time with one
// global atomic (a per-step atomic put an L2 round trip on every step of the critical path);
// the host sorts the log into the reference's loop order (report.py) and drops the unused
// tail records of each chunk (gi = -1, written at the end of the launch: close_log).
#define RSIM_LOG_CHUNK 32
__device__ __forceinline__ void log_step(const Params &P, FinBuf &F, int gi, i64 start, i64 end, i64 pre,
                                         i64 bs_after, i64 idx, int lane) {
    if (P.log != nullptr && lane == 0) {
        i64 n = F.lnext;
        if (n >= F.lend) { n = (i64)atomicAdd(P.log_n, (u64)RSIM_LOG_CHUNK); F.lend = n + RSIM_LOG_CHUNK; }
        F.lnext = n + 1;
        if (n < P.log_cap) {
            i64 *r = P.log + 6 * n;
            r[0] = gi; r[1] = start; r[2] = end; r[3] = pre; r[4] = bs_after; r[5] = idx;
        }
    }
}
__device__ __forceinline__ void close_log(const Params &P, FinBuf &F, int lane) {
    __syncwarp();
    if (P.log != nullptr)
        for (i64 n = F.lnext + lane; n < F.lend; n += 32)
            if (n < P.log_cap) P.log[6 * n] = -1;
    __syncwarp();
    if (lane == 0) F.lnext = F.lend = 0;
}

// Run the pending commit touch + pin of F (if any).
__device__ __noinline__ void run_touch_pin(const Params &P, FinBuf &F, int lane, int *werr_sm) {
    __syncwarp();
    const Table T = table_of(P, F.tpgi);
    u64 kk0[4];
    int sl[4];
    const bool slots = F.tpsl != nullptr && F.tpsp->tabver == F.tpver;   // no key moved since the probe
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const int j = 32 * q + lane;
        kk0[q] = j < min(F.tph, 128) ? F.tpkeys[j] : 0;
        sl[q] = (slots && j < min(F.tph, 128)) ? F.tpsl[j] : -1;
    }
    int werr = 0;
    warp_touch_pin(T, P.ckeys + F.tpa, kk0, slots ? sl : nullptr, F.tph, F.tpt, lane, werr);
    __syncwarp();
    if (lane == 0) {
        F.tpn = 0;
        if (werr && *werr_sm == 0) *werr_sm = werr;
    }
    __syncwarp();
}

__device__ __forceinline__ void flush_touch_pin(const Params &P, FinBuf &F, int lane, int *werr_sm, int gi = -1) {
    if (F.tpn && (gi < 0 || gi == F.tpgi)) run_touch_pin(P, F, lane, werr_sm);
}

// Finisher batch of one step (engine.py:357-361 for every finisher in F): runs
// on a register copy of the instance and writes back the KV$-side fields only
// (the step owns the engine-side fields). Out of line: finishes are rare.
__device__ __noinline__ void finish_batch(const Params &P, Inst *sp, int gi, FinBuf &F, int nf, i64 end, int lane,
                                          int *werr_sm) {
    flush_touch_pin(P, F, lane, werr_sm, gi);                      // eviction reads touch and pins
    int werr = *werr_sm;
    __syncwarp();
    if (lane == 0) werr_sm[1] += 1;                               // WarpBuf.fins (follows werr)
    Inst s = *sp;
    flush_finishers(P, gi, s, F, nf, end, lane, werr);
    __syncwarp();
    if (lane == 0) {
        sp->occ = s.occ; sp->tabver = s.tabver;
        sp->r_head = s.r_head; sp->r_tail = s.r_tail; sp->r_tailT = s.r_tailT;
        if (werr) *werr_sm = werr;
    }
    __syncwarp();
}

// Append the finishers of lane mask fm (lane l's request record at e) to F in
// lane order -- the reference's order within one ballot -- flushing F first if
// it would overflow.
// Deferral of finisher cache work past the publish of the decision being
// scored. The probe only needs the key *set* of the instance's table, and
// inserting whole chains (no eviction) changes the longest present prefix of
// the scored request R in a closed form: the table is prefix-closed along R's
// chain, a finished chain X contributes exactly its common prefix with R, so
//     h' = max(h, LCP(X, R))          (chain keys are equal iff prefixes are).
// So when no eviction can follow (occupancy + inserted keys <= capacity) and
// the instance's probe-ahead hit h is valid, the batch is parked in F and only
// h is raised; the caller applies the batch right after publishing.
struct Defer {
    const u64 *rkeys;    // the scored request's first 128 chain keys (shared memory)
    int rB;              // its prefix blocks
    int *hit;            // per local instance: probe-ahead hit blocks of the scored request
    u32 valid;           // instances whose probe-ahead hit is valid
    u32 moved;           // out: instances whose hit a parked batch raised (their probe slots are stale)
};

__device__ __forceinline__ void apply_deferred(const Params &P, FinBuf &F, int lane, int *werr_sm, Defer *df = nullptr) {
    if (F.dnf) {
        // the instance's probe-ahead hit no longer matches its table version: no more parking for it
        if (df != nullptr) df->valid &= ~(1u << F.dsi);
        finish_batch(P, F.dsp, F.dgi, F, F.dnf, F.dend, lane, werr_sm);
        __syncwarp();
        if (lane == 0) F.dnf = 0;
        __syncwarp();
    }
}

__device__ __forceinline__ void add_finishers(const Params &P, Inst *sp, int gi, FinBuf &F, int &nf, u32 fm,
                                              const Ent *e, i64 end, int lane, int *werr_sm, Defer *df) {
    if (nf == 0) apply_deferred(P, F, lane, werr_sm, df);         // F is about to be reused
    const int cnt = __popc(fm);
    if (nf + cnt > 32) { finish_batch(P, sp, gi, F, nf, end, lane, werr_sm); nf = 0; }
    const bool fin = (fm >> lane) & 1u;
    const int pos = nf + __popc(fm & lanemask_lt());
    int L = 0;
    if (fin) {
        F.a[pos] = e->a; F.oa[pos] = e->oa; F.B[pos] = e->B; F.hb[pos] = e->hb; F.kx[pos] = e->kx;
        L = e->L;
        F.L[pos] = L;
    }
    const int prev = nf == 0 ? 0 : F.pre[nf];
    const int incl = warp_incl_scan(L, lane);
    __syncwarp();
    if (lane == 0 && nf == 0) F.pre[0] = 0;
    if (fin) F.pre[pos + 1] = prev + incl;
    nf += cnt;
    __syncwarp();
}

// LCP of finisher f's full chain with the scored request, or -1 if it is not
// decidable from the first 128 depths.
__device__ __forceinline__ int chain_lcp(const Params &P, const FinBuf &F, int f, const Defer &df, int lane) {
    const int B = F.B[f], L = F.L[f];
    const int m = min(L, df.rB), mc = min(m, 128);
    int lcp = mc;
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const int j = 32 * q + lane;
        bool ne = false;
        if (j < mc) {
            const u64 xk = j < B ? P.ckeys[F.a[f] + j] : P.okeys[F.oa[f] + j - B];
            ne = xk != df.rkeys[j];
        }
        const u32 nm = __ballot_sync(FULL, ne);
        if (nm && lcp == mc) lcp = 32 * q + __ffs(nm) - 1;
    }
    if (lcp == 128 && m > 128) return -1;
    return lcp;
}

__device__ __forceinline__ void finish_or_defer(const Params &P, Inst *sp, int gi, int s, FinBuf &F, int nf, i64 end,
                                                int lane, int *werr_sm, Defer *df) {
    if (df != nullptr && ((df->valid >> s) & 1u) && F.dnf == 0 && (P.cap < 0 || sp->occ + F.pre[nf] <= P.cap)) {
        int h = df->hit[s];
        bool ok = true;
        for (int f = 0; f < nf && ok; f++) {
            // LCP(X, R) > h needs X.key[h] == R.key[h]. X's admission-hit keys X.key[0..hb) are
            // present (pinned by X until this finish) while R.key[h] is not, so h < hb rules it
            // out; otherwise it needs X.key[hb] == R.key[hb] (Ent.kx). Only then load X's chain.
            const int hbx = F.hb[f], m = min(F.L[f], df->rB);
            if (m <= h || h < hbx || hbx >= m) continue;           // cannot raise h
            if (F.kx[f] != 0 && hbx < 128 && F.kx[f] != df->rkeys[hbx]) continue;
            const int l = chain_lcp(P, F, f, *df, lane);
            if (l < 0) ok = false;
            else if (l > h) h = l;
        }
        if (ok) {
            const bool raised = h != df->hit[s];                   // lane-uniform
            if (raised) df->moved |= 1u << s;                       // (df is per-lane: every lane updates)
            __syncwarp();
            if (lane == 0) {
                if (raised) df->hit[s] = h;
                F.dnf = nf; F.dgi = gi; F.dsi = s; F.dend = end; F.dsp = sp; F.npark += 1;
            }
            __syncwarp();
            return;
        }
    }
    finish_batch(P, sp, gi, F, nf, end, lane, werr_sm);
}

// One engine step of instance gi starting at its next_step (form_batch +
// execute_batch, engine.py:291-355). Returns false if the plan was empty (the
// instance went idle). Queue/running records are read field by field from
// their (L1-resident) lines instead of being held in registers, so the step
// needs few registers; lane-uniform engine fields live in registers and go
// back to shared memory at the end. F is this warp's finisher buffer.
#ifdef RSIM_STEP_PROFILE
#define SP_MARK(i) do { const long long _t = clock64(); spc[i] += _t - spt; spt = _t; } while (0)
#else
#define SP_MARK(i) do { } while (0)
#endif
__device__ __forceinline__ bool inst_step_body(const Params &P, Inst *sp, int gi, int s, int lane, int *werr_sm,
                                               FinBuf &F, Defer *df) {
#ifdef RSIM_STEP_PROFILE
    long long spc[8] = {0, 0, 0, 0, 0, 0, 0, 0}, spt = clock64();
#endif
    const i64 t = sp->next_step;
    if (sp->due <= t) {                                            // form_batch flush, engine.py:293
        __syncwarp();
        if (lane == 0) flush_view(*sp, t);
        __syncwarp();
    }
    const int ndec = sp->r;                                        // running <= max_batch always
    const int q = sp->q, qh = sp->q_head;
    const i64 step_idx = sp->step_idx;
    const bool fin_step = ndec > 0 && sp->next_finish == step_idx;
    const i64 budget = P.chunk - ndec > 0 ? P.chunk - ndec : 0;   // engine.py:296
    const i64 slots = P.max_batch - ndec;                          // engine.py:297
    QEnt *qb = P.qbuf + ((size_t)gi << P.qlog2);
    REnt *rb = rlist(P, gi);
    const u32 qmask = (1u << P.qlog2) - 1u;
    SP_MARK(0);
    if (q == 0 && !fin_step && ndec > 0) {
        // pure decode step: no prefill, no pop, no finish (the general path below reduces to this)
        const i64 dcs0 = sp->dcs;
        const i64 end = t + decode_cost_us(P, ndec, dcs0);
        __syncwarp();
        if (lane == 0) {
            sp->total += ndec;
            sp->dcs = dcs0 + ndec;
            sp->busy_until = end;                                  // engine.py:349-352
            sp->due = end;
            sp->next_step = end;
            sp->step_idx = step_idx + 1;
        }
        log_step(P, F, gi, t, end, 0, (i64)ndec, step_idx, lane);
        __syncwarp();
        SP_MARK(7);
#ifdef RSIM_STEP_PROFILE
        if (P.ctr != nullptr && lane == 0) {
            long long tot = 0;
            for (int i = 0; i < 8; i++) { atomicAdd(P.ctr + 16 + i, (u64)spc[i]); tot += spc[i]; }
            atomicAdd(P.ctr + 28, (u64)1);                         // [28..29]: pure decode steps
            atomicAdd(P.ctr + 29, (u64)tot);
        }
#endif
        return true;
    }
    if (q == 0 && fin_step && ndec <= 32) {
        // decode step with finishes and at most 32 running (engine.py:333-347): one record per
        // lane; 32-bit warp reductions (REDUX) replace the 64-bit shuffle trees
        REnt *e = rb + lane;
        const bool valid = lane < ndec;
        const i64 v = valid ? e->v : RSIM_NONE;
        const i64 dcs0 = sp->dcs;
        const i64 end = t + decode_cost_us(P, ndec, dcs0);
        const bool fin = valid && v == step_idx;
        const bool keep = valid && !fin;
        const u32 fm = __ballot_sync(FULL, fin), km = __ballot_sync(FULL, keep);
        u64 g = 0;                                                 // in + out of a finisher (< 2^41)
        if (fin) { g = (u64)e->in + (u64)(u32)e->out; P.finish[e->req] = end; }
        const u64 gone = ((u64)__reduce_add_sync(FULL, (u32)(g >> 20)) << 20) + __reduce_add_sync(FULL, (u32)(g & 0xfffffu));
        int nf = 0;
        add_finishers(P, sp, gi, F, nf, fm, e, end, lane, werr_sm, df);
        const int dst = __popc(km & lanemask_lt());
        const bool move = keep && dst != lane;
        if (__any_sync(FULL, move)) {                              // compact: all reads before any write
            const ulonglong2 *src = reinterpret_cast<const ulonglong2 *>(e);
            const ulonglong2 z = make_ulonglong2(0ULL, 0ULL);
            const ulonglong2 c0 = move ? src[0] : z, c1 = move ? src[1] : z;   // unconditional: registers
            const ulonglong2 c2 = move ? src[2] : z, c3 = move ? src[3] : z;
            __syncwarp();
            if (move) {
                ulonglong2 *d = reinterpret_cast<ulonglong2 *>(rb + dst);
                d[0] = c0; d[1] = c1; d[2] = c2; d[3] = c3;
            }
        }
        const u32 mo = __reduce_min_sync(FULL, keep ? (u32)(v - step_idx) : 0xffffffffu);
        const i64 nfin = mo == 0xffffffffu ? RSIM_NONE : step_idx + (i64)mo;
        const int r = __popc(km);
        if (nf) finish_or_defer(P, sp, gi, s, F, nf, end, lane, werr_sm, df);
        __syncwarp();
        if (lane == 0) {
            sp->r = r;
            sp->total = sp->total + ndec - (i64)gone;
            sp->dcs = dcs0 + ndec - (i64)gone;
            sp->next_finish = nfin;
            sp->busy_until = end;                                  // engine.py:349-352
            sp->due = end;
            sp->next_step = end;
            sp->step_idx = step_idx + 1;
        }
        log_step(P, F, gi, t, end, 0, (i64)r, step_idx, lane);
        __syncwarp();
        SP_MARK(7);
#ifdef RSIM_STEP_PROFILE
        if (P.ctr != nullptr && lane == 0) {
            long long tot = 0;
            for (int i = 0; i < 8; i++) { atomicAdd(P.ctr + 16 + i, (u64)spc[i]); tot += spc[i]; }
            atomicAdd(P.ctr + 24, (u64)1);
            atomicAdd(P.ctr + 25, (u64)tot);
        }
#endif
        return true;
    }
    if (q == 1 && !fin_step) {
        // one queued request, no decode finish: the FIFO plan, pop and join of the general path
        // below for a single entry, on lane 0 (no warp scans); a pop that finishes at once
        // (out == 1) takes the general path
        QEnt *e = qb + (qh & qmask);
        const i64 budget0 = budget, slots0 = slots;
        int go = 0;
        i64 ptok1 = 0, end1 = 0, pre1 = 0, dcs1 = 0, tot1 = 0, nfin1 = 0;
        int r1 = 0, npop1 = 0;
        if (lane == 0) {
            const bool cached = sp->qcpos == (i64)qh;
            const ulonglong2 *src = reinterpret_cast<const ulonglong2 *>(cached ? &sp->qhead : e);
            ulonglong2 c0 = src[0], c1 = src[1], c2 = src[2], c3 = src[3];
            const i64 p = (i64)c0.x, in = (i64)c0.y;
            const int req = (int)(u32)c2.x, flags = (int)(u32)(c2.x >> 32), out = (int)(u32)c2.y;
            const bool alloc = slots0 > 0 && budget0 > 0;
            const i64 take = alloc ? (budget0 < p ? budget0 : p) : 0;
            const bool pop = alloc && p - take == 0;
            go = (alloc || ndec > 0) && !(pop && out == 1);
            if (go) {
                ptok1 = take;
                dcs1 = sp->dcs;
                pre1 = prefill_cost_us(P, ptok1);
                end1 = t + pre1 + decode_cost_us(P, ndec, dcs1);
                if (alloc && !(flags & 1)) P.first_sched[req] = t;
                tot1 = sp->total + (pop ? 1 : 0) + ndec;
                dcs1 += ndec;
                r1 = ndec;
                nfin1 = sp->next_finish;
                if (alloc && !pop) {                              // partial prefill: stays queued
                    c0.x = (u64)(p - take);
                    c2.x = (c2.x & 0xffffffffULL) | ((u64)(u32)(flags | 1) << 32);
                    ulonglong2 *dq = reinterpret_cast<ulonglong2 *>(e);
                    dq[0] = c0; dq[2] = c2;
                    ulonglong2 *dc = reinterpret_cast<ulonglong2 *>(&sp->qhead);
                    dc[0] = c0; dc[1] = c1; dc[2] = c2; dc[3] = c3;
                    sp->qcpos = qh;
                }
                if (pop) {                                        // first token; joins the running list
                    npop1 = 1;
                    P.first_token[req] = end1;
                    const i64 fstep = step_idx + out - 1;
                    c0.x = (u64)fstep;
                    ulonglong2 *d = reinterpret_cast<ulonglong2 *>(rb + r1);
                    d[0] = c0; d[1] = c1; d[2] = c2; d[3] = c3;
                    dcs1 += in + 1;
                    r1 += 1;
                    nfin1 = fstep < nfin1 ? fstep : nfin1;
                }
                sp->q_head = (qh + npop1) & (int)qmask;
                sp->q = 1 - npop1;
                sp->r = r1;
                sp->pend -= ptok1;
                sp->total = tot1;
                sp->dcs = dcs1;
                sp->next_finish = nfin1;
                sp->busy_until = end1;                             // engine.py:349-352
                sp->due = end1;
                sp->next_step = end1;
                sp->step_idx = step_idx + 1;
            }
        }
        go = __shfl_sync(FULL, go, 0);
        if (go) {
            if (P.log != nullptr) {
                end1 = __shfl_sync(FULL, end1, 0); pre1 = __shfl_sync(FULL, pre1, 0);
                r1 = __shfl_sync(FULL, r1, 0); npop1 = __shfl_sync(FULL, npop1, 0);
                log_step(P, F, gi, t, end1, pre1, (i64)(1 - npop1) + r1, step_idx, lane);
            }
            __syncwarp();
            SP_MARK(7);
#ifdef RSIM_STEP_PROFILE
            if (P.ctr != nullptr && lane == 0) {
                long long tot = 0;
                for (int i = 0; i < 8; i++) { atomicAdd(P.ctr + 16 + i, (u64)spc[i]); tot += spc[i]; }
                atomicAdd(P.ctr + 26, (u64)1);
                atomicAdd(P.ctr + 27, (u64)tot);
            }
#endif
            return true;
        }
    }

    if (q > 0) {                                                   // the general path rewrites heads
        __syncwarp();
        if (lane == 0) sp->qcpos = -1;
        __syncwarp();
    }
    // pass 1: FIFO plan (_plan_allocations, engine.py:174-184). Entry j is
    // allocated iff j < slots and the budget left before it is positive.
    i64 ptok = 0, v0 = 0;
    int nalloc = 0;
    {
        i64 cum = 0;
        for (int j0 = 0; j0 < q && j0 < slots && cum < budget; j0 += 32) {
            const int j = j0 + lane;
            const bool valid = j < q && j < slots;
            const i64 p = valid ? qb[(qh + j) & qmask].v : 0;
            if (j0 == 0) v0 = p;
            const i64 incl = warp_incl_scan(p, lane);
            const i64 excl = cum + incl - p;
            const bool alloc = valid && excl < budget;
            const i64 take = alloc ? min(budget - excl, p) : 0;
            const int na = __popc(__ballot_sync(FULL, alloc));
            nalloc += na;
            ptok += warp_sum(take);
            cum += __shfl_sync(FULL, incl, 31);
            if (na < 32) break;
        }
    }
    if (nalloc == 0 && ndec == 0) {                                // empty plan: instance goes idle
        __syncwarp();
        if (lane == 0) sp->next_step = RSIM_NONE;
        __syncwarp();
        return false;
    }
    SP_MARK(1);
    i64 dcs = sp->dcs;
    const i64 pre = prefill_cost_us(P, ptok);
    const i64 end = t + pre + decode_cost_us(P, ndec, dcs);       // ctx = sum(in+gen) over decode = dcs
    SP_MARK(2);

    // pass 2: apply allocations (engine.py:314-319); pops = allocated entries
    // left with pending == 0 (a prefix of the allocation)
    int npop = 0;
    {
        i64 cum = 0;
        for (int j0 = 0; j0 < nalloc; j0 += 32) {
            const int j = j0 + lane;
            const bool alloc = j < nalloc;
            QEnt *e = qb + ((qh + j) & qmask);
            const i64 p = alloc ? (j0 == 0 ? v0 : e->v) : 0;
            const i64 incl = warp_incl_scan(p, lane);
            const i64 excl = cum + incl - p;
            const i64 take = alloc ? min(budget - excl, p) : 0;
            if (alloc) {
                const int flags = e->flags;
                if (!(flags & 1)) P.first_sched[e->req] = t;
                if (p - take != 0) { e->v = p - take; e->flags = flags | 1; }   // a popped record is consumed as is
            }
            npop += __popc(__ballot_sync(FULL, alloc && p - take == 0));
            cum += __shfl_sync(FULL, incl, 31);
        }
    }
    i64 total = sp->total + npop;
    int nf = 0;
    SP_MARK(3);

    // queue heads with pending == 0 get their first token (engine.py:321-331);
    // out == 1 finishes right away, in pop order.
    for (int j0 = 0; j0 < npop; j0 += 32) {
        const int j = j0 + lane;
        const bool pop = j < npop;
        const QEnt *e = qb + ((qh + j) & qmask);
        bool fin = false;
        if (pop) {
            const int req = e->req;
            P.first_token[req] = end;
            fin = e->out == 1;
            if (fin) P.finish[req] = end;
        }
        const u32 fm = __ballot_sync(FULL, fin);
        if (fm) {
            total -= warp_sum(fin ? e->in + 1 : (i64)0);
            add_finishers(P, sp, gi, F, nf, fm, e, end, lane, werr_sm, df);
        }
    }

    SP_MARK(4);
    // decode (engine.py:333-347): every running request gains a token; those
    // whose finish step is now leave in running order.
    total += ndec;
    dcs += ndec;
    int r = ndec;
    i64 nfin = sp->next_finish;
    if (fin_step) {
        int w = 0;
        i64 nf_step = RSIM_NONE;
        for (int j0 = 0; j0 < ndec; j0 += 32) {
            const int j = j0 + lane;
            const bool valid = j < ndec;
            REnt *e = rb + j;
            const i64 v = valid ? e->v : RSIM_NONE;
            const bool fin = valid && v == step_idx;
            const bool keep = valid && !fin;
            const u32 km = __ballot_sync(FULL, keep);
            const int dst = w + __popc(km & lanemask_lt());
            const bool move = keep && dst != j;
            if (keep) nf_step = v < nf_step ? v : nf_step;
            const u32 fm = __ballot_sync(FULL, fin);
            if (fm) {
                i64 gone = 0;
                if (fin) { gone = e->in + e->out; P.finish[e->req] = end; }   // generated == out at finish
                gone = warp_sum(gone);
                dcs -= gone;
                total -= gone;
                add_finishers(P, sp, gi, F, nf, fm, e, end, lane, werr_sm, df);
            }
            if (__any_sync(FULL, move)) {                  // compact: all reads of this chunk before any write
                const ulonglong2 *src = reinterpret_cast<const ulonglong2 *>(e);
                const ulonglong2 z = make_ulonglong2(0ULL, 0ULL);
                const ulonglong2 c0 = move ? src[0] : z, c1 = move ? src[1] : z;
                const ulonglong2 c2 = move ? src[2] : z, c3 = move ? src[3] : z;
                __syncwarp();
                if (move) {
                    ulonglong2 *d = reinterpret_cast<ulonglong2 *>(rb + dst);
                    d[0] = c0; d[1] = c1; d[2] = c2; d[3] = c3;
                }
            }
            __syncwarp();
            w += __popc(km);
        }
        r = w;
        nfin = warp_min_i64(nf_step);
    }
    SP_MARK(5);
    if (nf) finish_or_defer(P, sp, gi, s, F, nf, end, lane, werr_sm, df);
    SP_MARK(6);

    // popped requests with out > 1 join the running list (after the removals)
    for (int j0 = 0; j0 < npop; j0 += 32) {
        const int j = j0 + lane;
        const bool pop = j < npop;
        const QEnt *e = qb + ((qh + j) & qmask);
        const int out = pop ? e->out : 0;
        const bool join = pop && out > 1;
        const u32 jm = __ballot_sync(FULL, join);
        i64 din = 0;
        if (join) {
            const ulonglong2 *src = reinterpret_cast<const ulonglong2 *>(e);
            ulonglong2 c0 = src[0], c1 = src[1], c2 = src[2], c3 = src[3];
            const i64 fstep = step_idx + out - 1;
            din = (i64)c0.y + 1;                           // in + 1
            c0.x = (u64)fstep;                             // v = finish step
            ulonglong2 *d = reinterpret_cast<ulonglong2 *>(rb + r + __popc(jm & lanemask_lt()));
            d[0] = c0; d[1] = c1; d[2] = c2; d[3] = c3;
            nfin = fstep < nfin ? fstep : nfin;
        }
        dcs += warp_sum(din);
        r += __popc(jm);
    }
    if (npop) nfin = warp_min_i64(nfin);

    __syncwarp();
    if (lane == 0) {
        sp->q_head = (qh + npop) & (int)qmask;
        sp->q = q - npop;
        sp->r = r;
        sp->pend -= ptok;
        sp->total = total;
        sp->dcs = dcs;
        sp->next_finish = nfin;
        sp->busy_until = end;                                      // engine.py:349-352
        sp->due = end;
        sp->next_step = end;
        sp->step_idx = step_idx + 1;
    }
    log_step(P, F, gi, t, end, pre, (i64)(q - npop) + r, step_idx, lane);
    __syncwarp();
    SP_MARK(7);
#ifdef RSIM_STEP_PROFILE
    if (P.ctr != nullptr && lane == 0) {
        long long tot = 0;
        for (int i = 0; i < 8; i++) { atomicAdd(P.ctr + 16 + i, (u64)spc[i]); tot += spc[i]; }
        const int kind = fin_step ? 0 : 1;                         // [24..27]: finishing / other full steps
        atomicAdd(P.ctr + 24 + 2 * kind, (u64)1);
        atomicAdd(P.ctr + 25 + 2 * kind, (u64)tot);
    }
#endif
    return true;
}

// Entry used by the replay loop (counts SM cycles in engine steps when profiling).
__device__ __forceinline__ bool inst_step(const Params &P, Inst *sp, int gi, int s, int lane, int *werr_sm, FinBuf &F,
                                          Defer *df) {
    const long long c0 = clock64();
    const bool ran = inst_step_body(P, sp, gi, s, lane, werr_sm, F, df);
    if (P.ctr != nullptr && lane == 0) atomicAdd(P.ctr + 2, (u64)(clock64() - c0));   // SM cycles in engine steps
    return ran;
}
