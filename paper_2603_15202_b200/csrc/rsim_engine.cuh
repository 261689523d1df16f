// rsim_engine.cuh -- one instance's engine step, executed by its owning warp.
//
// Restates InstanceSim.form_batch + execute_batch (reference engine.py:291-355)
// with the cost model of engine.py:81-96, on the instance's state held in
// shared memory. FIFO chunked-prefill allocation is a warp prefix sum over
// the queue head; decode bookkeeping is O(1) per step because each running
// request's finish step is known when it joins (finish = join + out - 1), so
// the running list is only scanned on steps where something finishes.
#pragma once
#include "rsim_cache.cuh"

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

// _finish (engine.py:357-372): unpin the admission hit, insert the full
// prefix+output chain stamped with the step end, evict down to capacity.
__device__ void finish_cache(const Params &P, int gi, i64 &occ, int req, i64 end, int lane, int &werr) {
    Table T = table_of(P, gi);
    const i64 a = P.blk_off[req];
    const int B = (int)(P.blk_off[req + 1] - a);
    const i64 oa = P.ooff[req];
    const int L = B + (int)(P.ooff[req + 1] - oa);
    occ += warp_unpin_insert(T, P.ckeys + a, B, P.okeys + oa, L, P.hit_blocks[req], end, lane, werr);
    if (occ > P.max_occ) werr = DEV_E_TABLE_FULL;
    if (P.cap >= 0 && occ > P.cap && !werr) warp_evict(T, P.cap, occ, lane, werr);
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
// the plan was empty (the instance went idle).
__device__ bool inst_step(const Params &P, Inst *sp, int gi, int lane, int &werr) {
    Inst s = *sp;
    const i64 t = s.next_step;
    flush_view(s, t);                                              // form_batch flush, engine.py:293
    const int ndec = s.r;                                          // running <= max_batch always
    const i64 budget = P.chunk - ndec > 0 ? P.chunk - ndec : 0;   // engine.py:296
    const i64 slots = P.max_batch - ndec;                          // engine.py:297
    QEnt *qb = P.qbuf + ((size_t)gi << P.qlog2);
    const u32 qmask = (1u << P.qlog2) - 1u;

    // pass 1: FIFO plan (_plan_allocations, engine.py:174-184). Entry j is
    // allocated iff j < slots and the budget left before it is positive.
    i64 ptok = 0;
    int nalloc = 0;
    {
        i64 cum = 0;
        for (int j0 = 0; j0 < s.q && j0 < slots && cum < budget; j0 += 32) {
            int j = j0 + lane;
            bool valid = j < s.q && j < slots;
            i64 p = valid ? qb[(s.q_head + j) & qmask].pending : 0;
            i64 incl = warp_incl_scan(p, lane);
            i64 excl = cum + incl - p;
            bool alloc = valid && excl < budget;
            i64 take = alloc ? min(budget - excl, p) : 0;
            int na = __popc(__ballot_sync(FULL, alloc));
            i64 ts = warp_sum(take);
            nalloc += na; ptok += ts;
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

    // pass 2: apply allocations (engine.py:314-319)
    int npop = 0;
    {
        i64 cum = 0;
        for (int j0 = 0; j0 < nalloc; j0 += 32) {
            int j = j0 + lane;
            bool alloc = j < nalloc;
            QEnt e;
            e.pending = 0; e.req = 0; e.flags = 0;
            if (alloc) e = qb[(s.q_head + j) & qmask];
            i64 p = alloc ? e.pending : 0;
            i64 incl = warp_incl_scan(p, lane);
            i64 excl = cum + incl - p;
            i64 take = alloc ? min(budget - excl, p) : 0;
            if (alloc) {
                if (!(e.flags & 1)) P.first_sched[e.req] = t;
                e.pending = p - take;
                e.flags |= 1;
                qb[(s.q_head + j) & qmask] = e;
            }
            npop += __popc(__ballot_sync(FULL, alloc && e.pending == 0));
            cum += __shfl_sync(FULL, incl, 31);
        }
    }
    s.pend -= ptok;
    __syncwarp();

    // queue heads with pending == 0 get their first token (engine.py:321-331);
    // out == 1 finishes right away, in pop order.
    const int head0 = s.q_head;
    s.total += npop;
    for (int j0 = 0; j0 < npop; j0 += 32) {
        int j = j0 + lane;
        bool pop = j < npop;
        int req = pop ? qb[(head0 + j) & qmask].req : 0;
        i64 out = pop ? P.out_tok[req] : 0;
        if (pop) P.first_token[req] = end;
        u32 fm = __ballot_sync(FULL, pop && out == 1);
        while (fm) {
            int l = __ffs(fm) - 1;
            fm &= fm - 1;
            int rq = __shfl_sync(FULL, req, l);
            if (lane == 0) P.finish[rq] = end;
            s.total -= P.in_tok[rq] + 1;
            if (!werr) finish_cache(P, gi, s.occ, rq, end, lane, werr);
        }
    }
    s.q_head = (s.q_head + npop) & (int)qmask;
    s.q -= npop;

    // decode (engine.py:333-347): every running request gains a token; those
    // whose finish step is now leave in running order.
    REnt *rb = P.rbuf + (size_t)gi * (size_t)P.max_batch;
    s.total += ndec;
    s.dcs += ndec;
    if (ndec > 0 && s.next_finish == s.step_idx) {
        int w = 0;
        i64 nf = RSIM_NONE;
        for (int j0 = 0; j0 < ndec; j0 += 32) {
            int j = j0 + lane;
            bool valid = j < ndec;
            REnt e;
            e.req = 0; e.pad = 0; e.finish_step = 0;
            if (valid) e = rb[j];
            __syncwarp();
            bool fin = valid && e.finish_step == s.step_idx;
            bool keep = valid && !fin;
            u32 km = __ballot_sync(FULL, keep);
            if (keep) {
                rb[w + __popc(km & lanemask_lt())] = e;
                nf = e.finish_step < nf ? e.finish_step : nf;
            }
            w += __popc(km);
            u32 fm = __ballot_sync(FULL, fin);
            while (fm) {
                int l = __ffs(fm) - 1;
                fm &= fm - 1;
                int rq = __shfl_sync(FULL, e.req, l);
                i64 gone = P.in_tok[rq] + P.out_tok[rq];        // generated == out at finish
                if (lane == 0) P.finish[rq] = end;
                s.dcs -= gone;
                s.total -= gone;
                if (!werr) finish_cache(P, gi, s.occ, rq, end, lane, werr);
            }
            __syncwarp();
        }
        s.r = w;
        s.next_finish = warp_min_i64(nf);
    }

    // popped requests with out > 1 join the running list (after the removals)
    {
        i64 nf = s.next_finish;
        for (int j0 = 0; j0 < npop; j0 += 32) {
            int j = j0 + lane;
            bool pop = j < npop;
            int req = pop ? qb[(head0 + j) & qmask].req : 0;
            i64 out = pop ? P.out_tok[req] : 0;
            bool join = pop && out > 1;
            u32 jm = __ballot_sync(FULL, join);
            i64 fs = s.step_idx + out - 1;
            if (join) {
                REnt e;
                e.req = req; e.pad = 0; e.finish_step = fs;
                rb[s.r + __popc(jm & lanemask_lt())] = e;
                nf = fs < nf ? fs : nf;
            }
            s.dcs += warp_sum(join ? P.in_tok[req] + 1 : (i64)0);
            s.r += __popc(jm);
        }
        s.next_finish = warp_min_i64(nf);
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
