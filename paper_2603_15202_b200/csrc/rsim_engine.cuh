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

__device__ __forceinline__ void flush_view(Inst &s, i64 now) {   // engine.py:240-246
    if (s.due <= now) {
        s.v_r = s.r; s.v_q = s.q; s.v_pend = s.pend; s.v_total = s.total; s.v_dc = s.dcs;
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
    s.occ += warp_unpin_insert(T, P.ckeys + a, B, P.okeys + oa, L, hb, end, lane, werr);
    if (s.occ > P.max_occ) werr = DEV_E_TABLE_FULL;
    evict_to_capacity(P, T, s, gi, lane, werr);
}

// Process the finishers collected in F, in collection order (= the reference's:
// queue-pop finishes, then decode finishes in running order). When no eviction
// can happen before the last insert, all chains go in one batched pass.
__device__ void flush_finishers(const Params &P, int gi, Inst &s, FinBuf &F, int nf, i64 end, int lane, int &werr) {
    if (nf == 0 || werr) return;
    const long long c0 = clock64();
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

__device__ __forceinline__ void log_step(const Params &P, int gi, i64 start, i64 end, i64 pre, i64 bs_after,
                                         i64 idx, int lane) {
    if (P.log != nullptr && lane == 0) {
        u64 n = atomicAdd(P.log_n, 1ULL);
        if ((i64)n < P.log_cap) {
            i64 *r = P.log + 6 * n;
            r[0] = gi; r[1] = start; r[2] = end; r[3] = pre; r[4] = bs_after; r[5] = idx;
        }
    }
}

// One engine step of instance gi starting at s.next_step. Returns false if
// the plan was empty (the instance went idle). F is this warp's finisher buffer.
__device__ __forceinline__ bool inst_step_body(const Params &P, Inst *sp, int gi, int lane, int &werr, FinBuf &F) {
    Inst s = *sp;
    const i64 t = s.next_step;
    flush_view(s, t);                                              // form_batch flush, engine.py:293
    const int ndec = s.r;                                          // running <= max_batch always
    const i64 budget = P.chunk - ndec > 0 ? P.chunk - ndec : 0;   // engine.py:296
    const i64 slots = P.max_batch - ndec;                          // engine.py:297
    QEnt *qb = P.qbuf + ((size_t)gi << P.qlog2);
    REnt *rb = P.rbuf + (size_t)gi * (size_t)P.max_batch;
    const u32 qmask = (1u << P.qlog2) - 1u;
    const bool fin_step = ndec > 0 && s.next_finish == s.step_idx;
    // the running list's first 32 records load together with the queue head
    Ent r0;
    r0.v = RSIM_NONE;
    if (fin_step && lane < ndec) r0 = rb[lane];

    // pass 1: FIFO plan (_plan_allocations, engine.py:174-184). Entry j is
    // allocated iff j < slots and the budget left before it is positive.
    // The first 32 entries stay in registers for pass 2.
    i64 ptok = 0;
    int nalloc = 0;
    Ent e0;
    e0.v = 0;
    {
        i64 cum = 0;
        for (int j0 = 0; j0 < s.q && j0 < slots && cum < budget; j0 += 32) {
            const int j = j0 + lane;
            const bool valid = j < s.q && j < slots;
            Ent e;
            e.v = 0;
            if (valid) e = qb[(s.q_head + j) & qmask];
            if (j0 == 0) e0 = e;
            const i64 p = valid ? e.v : 0;
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
        s.next_step = RSIM_NONE;
        __syncwarp();
        if (lane == 0) *sp = s;
        __syncwarp();
        return false;
    }
    const i64 pre = prefill_cost_us(P, ptok);
    const i64 end = t + pre + decode_cost_us(P, ndec, s.dcs);      // ctx = sum(in+gen) over decode = dcs

    // pass 2: apply allocations (engine.py:314-319); pops = allocated entries
    // left with pending == 0 (a prefix of the allocation)
    int npop = 0;
    {
        i64 cum = 0;
        for (int j0 = 0; j0 < nalloc; j0 += 32) {
            const int j = j0 + lane;
            const bool alloc = j < nalloc;
            Ent e = e0;
            if (j0 > 0 && alloc) e = qb[(s.q_head + j) & qmask];
            const i64 p = alloc ? e.v : 0;
            const i64 incl = warp_incl_scan(p, lane);
            const i64 excl = cum + incl - p;
            const i64 take = alloc ? min(budget - excl, p) : 0;
            if (alloc) {
                if (!(e.flags & 1)) P.first_sched[e.req] = t;
                if (p - take != 0) {                        // a popped record is consumed below as is
                    Ent u = e;
                    u.v = p - take;
                    u.flags |= 1;
                    qb[(s.q_head + j) & qmask] = u;
                }
            }
            npop += __popc(__ballot_sync(FULL, alloc && p - take == 0));
            cum += __shfl_sync(FULL, incl, 31);
        }
    }
    s.pend -= ptok;
    __syncwarp();

    int nf = 0;
    auto add_fin = [&](const Ent &f) {
        if (nf == 32) { flush_finishers(P, gi, s, F, nf, end, lane, werr); nf = 0; }
        if (lane == 0) {
            if (nf == 0) F.pre[0] = 0;
            F.a[nf] = f.a; F.oa[nf] = f.oa; F.B[nf] = f.B; F.L[nf] = f.L; F.hb[nf] = f.hb;
            F.pre[nf + 1] = F.pre[nf] + f.L;
        }
        nf++;
    };

    // queue heads with pending == 0 get their first token (engine.py:321-331);
    // out == 1 finishes right away, in pop order.
    const int head0 = s.q_head;
    s.total += npop;
    for (int j0 = 0; j0 < npop; j0 += 32) {
        const int j = j0 + lane;
        const bool pop = j < npop;
        Ent e = e0;
        if (j0 > 0 && pop) e = qb[(head0 + j) & qmask];
        if (pop) P.first_token[e.req] = end;
        u32 fm = __ballot_sync(FULL, pop && e.out == 1);
        while (fm) {
            const int l = __ffs(fm) - 1;
            fm &= fm - 1;
            const Ent f = shfl_ent(e, l);
            if (lane == 0) P.finish[f.req] = end;
            s.total -= f.in + 1;
            add_fin(f);
        }
    }
    s.q_head = (s.q_head + npop) & (int)qmask;
    s.q -= npop;

    // decode (engine.py:333-347): every running request gains a token; those
    // whose finish step is now leave in running order.
    s.total += ndec;
    s.dcs += ndec;
    if (fin_step) {
        int w = 0;
        i64 nf_step = RSIM_NONE;
        for (int j0 = 0; j0 < ndec; j0 += 32) {
            const int j = j0 + lane;
            const bool valid = j < ndec;
            Ent e = r0;
            if (j0 > 0) { e.v = RSIM_NONE; if (valid) e = rb[j]; }
            __syncwarp();
            const bool fin = valid && e.v == s.step_idx;
            const bool keep = valid && !fin;
            const u32 km = __ballot_sync(FULL, keep);
            if (keep) {
                const int dst = w + __popc(km & lanemask_lt());
                if (dst != j) rb[dst] = e;
                nf_step = e.v < nf_step ? e.v : nf_step;
            }
            w += __popc(km);
            u32 fm = __ballot_sync(FULL, fin);
            while (fm) {
                const int l = __ffs(fm) - 1;
                fm &= fm - 1;
                const Ent f = shfl_ent(e, l);
                const i64 gone = f.in + f.out;                     // generated == out at finish
                if (lane == 0) P.finish[f.req] = end;
                s.dcs -= gone;
                s.total -= gone;
                add_fin(f);
            }
            __syncwarp();
        }
        s.r = w;
        s.next_finish = warp_min_i64(nf_step);
    }
    flush_finishers(P, gi, s, F, nf, end, lane, werr);

    // popped requests with out > 1 join the running list (after the removals)
    {
        i64 nfin = s.next_finish;
        for (int j0 = 0; j0 < npop; j0 += 32) {
            const int j = j0 + lane;
            const bool pop = j < npop;
            Ent e = e0;
            if (j0 > 0 && pop) e = qb[(head0 + j) & qmask];
            const bool join = pop && e.out > 1;
            const u32 jm = __ballot_sync(FULL, join);
            if (join) {
                e.v = s.step_idx + e.out - 1;
                rb[s.r + __popc(jm & lanemask_lt())] = e;
                nfin = e.v < nfin ? e.v : nfin;
            }
            s.dcs += warp_sum(join ? e.in + 1 : (i64)0);
            s.r += __popc(jm);
        }
        s.next_finish = warp_min_i64(nfin);
    }

    s.busy_until = end;                                            // engine.py:349-352
    s.due = end;
    s.next_step = end;
    log_step(P, gi, t, end, pre, (i64)s.q + s.r, s.step_idx, lane);
    s.step_idx += 1;
    __syncwarp();
    if (lane == 0) *sp = s;
    __syncwarp();
    return true;
}

// Non-inlined entry used by the replay loop: the error word lives in shared
// memory so no caller register has its address taken.
__device__ __noinline__ bool inst_step(const Params &P, Inst *sp, int gi, int lane, int *werr_sm, FinBuf &F) {
    int werr = *werr_sm;
    const long long c0 = clock64();
    const bool ran = inst_step_body(P, sp, gi, lane, werr, F);
    if (P.ctr != nullptr && lane == 0) atomicAdd(P.ctr + 2, (u64)(clock64() - c0));   // SM cycles in engine steps
    __syncwarp();
    if (lane == 0 && werr) *werr_sm = werr;
    __syncwarp();
    return ran;
}
