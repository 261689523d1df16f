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

// ---------------------------------------------------------------- K1
// One warp per 32 consecutive requests: their blocks are one contiguous CSR
// span, staged through shared memory with coalesced loads/stores; each lane
// folds its own request's chain (hashing.py:36-47; splitmix64 is not
// associative, so the chain is sequential per request). Output-block keys
// extend the chain with stable_key(0x0F0C0DE, rid, idx) (engine.py:363-372).
#define K1_WIN 256
#define K1_WARPS 8
__global__ void __launch_bounds__(32 * K1_WARPS)
k1_chain_keys(const i64 *__restrict__ blk_off, const u64 *__restrict__ blocks, u64 *__restrict__ ckeys,
              const i64 *__restrict__ ooff, u64 *__restrict__ okeys, const u64 *__restrict__ rid,
              i64 r0, i64 r1, u64 empty, int *flag) {
    __shared__ u64 sbuf[K1_WARPS][K1_WIN];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const i64 wid = (i64)blockIdx.x * K1_WARPS + wl;
    const i64 base = r0 + wid * 32;
    if (base >= r1) return;
    const i64 rlast = min(base + 32, r1);
    const i64 r = base + lane;
    const bool mine = r < rlast;
    const i64 a = mine ? blk_off[r] : 0, b = mine ? blk_off[r + 1] : 0;
    const i64 span0 = blk_off[base], span1 = blk_off[rlast];
    u64 acc = RSIM_GOLDEN;
    bool bad = false;
    u64 *sb = sbuf[wl];
    for (i64 ws = span0; ws < span1; ws += K1_WIN) {
        const i64 we = min(ws + K1_WIN, span1);
#pragma unroll
        for (int i = 0; i < K1_WIN / 32; i++) {
            i64 p = ws + i * 32 + lane;
            if (p < we) sb[i * 32 + lane] = __ldcs(blocks + p);
        }
        __syncwarp();
        const i64 lo = max(a, ws), hi = min(b, we);
        for (i64 j = lo; j < hi; j++) {
            acc = combine64(acc, sb[j - ws]);
            bad |= (acc == empty);
            sb[j - ws] = acc;
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < K1_WIN / 32; i++) {
            i64 p = ws + i * 32 + lane;
            if (p < we) __stcs(ckeys + p, sb[i * 32 + lane]);
        }
        __syncwarp();
    }
    if (mine) {
        const i64 o0 = ooff[r], o1 = ooff[r + 1];
        const u64 salt = combine64(combine64(RSIM_GOLDEN, RSIM_OUTPUT_SALT), rid[r]);
        for (i64 i = o0; i < o1; i++) {
            acc = combine64(acc, combine64(salt, (u64)(i - o0)));
            bad |= (acc == empty);
            okeys[i] = acc;
        }
    }
    if (__any_sync(FULL, bad) && lane == 0) atomicExch(flag, 1);
}

// ---------------------------------------------------------------- cluster PTX
__device__ __forceinline__ u32 cluster_ctarank() { u32 r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ u32 smem_addr(const void *p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void st_cluster_u64(u32 local_addr, u32 rank, u64 v) {
    u32 remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_addr), "r"(rank));
    asm volatile("st.shared::cluster.u64 [%0], %1;" :: "r"(remote), "l"(v) : "memory");
}

__device__ __forceinline__ u64 globaltimer() { u64 t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

struct __align__(16) Part { u64 minb; u32 cnt; u32 err; };

// ---------------------------------------------------------------- score
// Policy scores (policies.py:104-139) as IEEE doubles, bit-exact with
// CPython's float arithmetic (each op rounded to nearest, no contraction).
__device__ __forceinline__ double score_of(const Params &P, const Inst &s, int h, i64 in) {
    const i64 bsz = (i64)s.v_r + s.v_q;
    if (P.policy == 0) {                                            // multiplicative
        i64 ht = (i64)h * P.bs; if (ht > in) ht = in;
        i64 nw = in - ht; if (nw < 1) nw = 1;
        double kv = P.kv_ind == 0 ? __ll2double_rn(s.v_pend + nw)
                                  : __dsub_rn(1.0, __ddiv_rn(__ll2double_rn(ht), __ll2double_rn(in)));
        i64 bal = P.bal_ind == 0 ? bsz : s.v_total;
        return __dmul_rn(kv, __ll2double_rn(bal > 1 ? bal : 1));
    } else if (P.policy == 1) {                                     // vllm
        return __dadd_rn(__dmul_rn(P.qw, (double)s.v_q), (double)s.v_r);
    }
    return __ll2double_rn(bsz);                                     // least_bs
}

// enqueue on the winner (InstanceSim.enqueue, engine.py:262-289) + route bookkeeping
__device__ void commit(const Params &P, Inst *sp, int gi, i64 k, int h, i64 t, const u64 kk0[4], i64 in,
                       int lane, int &werr) {
    Table T = table_of(P, gi);
    warp_touch_pin(T, P.ckeys + P.blk_off[k], kk0, h, t, lane, werr);
    Inst s = *sp;
    i64 ht = (i64)h * P.bs; if (ht > in) ht = in;
    i64 pending = in - ht; if (pending < 1) pending = 1;
    if (s.q >= (1 << P.qlog2)) { werr = DEV_E_QUEUE_OVERFLOW; return; }
    if (lane == 0) {
        QEnt e; e.req = (int)k; e.flags = 0; e.pending = pending;
        P.qbuf[((size_t)gi << P.qlog2) + ((s.q_head + s.q) & ((1 << P.qlog2) - 1))] = e;
        P.hit_blocks[k] = h;
        P.chosen[k] = gi;
        P.hit_tokens[k] = ht;
        P.route_bs[k] = (i64)s.q + 1 + s.r;
    }
    s.q += 1; s.pend += pending; s.total += in;
    s.v_q += 1; s.v_pend += pending; s.v_total += in;              // view moves incrementally (engine.py:284-285)
    if (s.next_step == RSIM_NONE && s.busy_until <= t) s.next_step = t;   // cluster.py:284-285
    __syncwarp();
    if (lane == 0) *sp = s;
    __syncwarp();
}

enum { MODE_REPLAY = 0, MODE_DRAIN = 1, MODE_ROUTE = 2, MODE_ENQUEUE = 3 };

// ---------------------------------------------------------------- replay
// Persistent launch over a cluster of C CTAs (C <= 16, one instance shard per
// CTA, engine state in shared memory). Per decision: every warp drains and
// probes its own instances, warp partials meet in shared memory, CTA
// partials are pushed to every CTA of the cluster over DSMEM, one hardware
// cluster barrier, then every CTA derives the same global winner and the
// owning warp commits. No host round trip per decision.
#define RSIM_MAX_WARPS 16
__global__ void __launch_bounds__(32 * RSIM_MAX_WARPS, 1)
replay_kernel(Params P, i64 k0, i64 k1, i64 until, int mode, int target) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int C = P.C, W = P.W, ipw = P.ipw;
    const int cta = (C > 1) ? (int)cluster_ctarank() : 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int base = cta * P.per_cta;
    const int nloc = max(0, min(P.per_cta, P.N - base));
    Inst *st = (Inst *)smem;
    Part *wp = (Part *)(st + P.per_cta);      // [2][W]
    Part *cp = wp + 2 * W;                    // [2][C]

    // load this CTA's instance shard
    {
        const u64 *src = (const u64 *)(P.inst + base);
        u64 *dst = (u64 *)st;
        const int words = nloc * (int)(sizeof(Inst) / 8);
        for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
    }
    unsigned __int128 counter = ((unsigned __int128)P.tie[1] << 64) | P.tie[0];
    __syncthreads();
    if (C > 1) cluster_sync_all();

    const int l0 = warp * ipw;
    const int nmine = max(0, min(ipw, nloc - l0));
    int werr = 0;
    u64 c_bytes = 0, c_steps = 0;   // algorithmic probe bytes / engine steps of this warp

    if (mode == MODE_DRAIN) {
        for (int s = 0; s < nmine; s++) {
            Inst *sp = st + l0 + s;
            while (!werr && sp->next_step < until) c_steps += inst_step(P, sp, base + l0 + s, lane, werr);
        }
    } else {
        for (i64 k = k0; k < k1; k++) {
            const int par = (int)(k & 1);
            const i64 t = (mode == MODE_REPLAY) ? P.arrival[k] : until;
            // ---- K4: advance my instances through steps starting before t (cluster.py:250-273)
            if (mode == MODE_REPLAY) {
                for (int s = 0; s < nmine; s++) {
                    Inst *sp = st + l0 + s;
                    while (!werr && sp->next_step < t) c_steps += inst_step(P, sp, base + l0 + s, lane, werr);
                }
            }
            // ---- K2: flush views, probe, score (cluster.py:106-128, policies.py:117-139)
            const i64 a = P.blk_off[k];
            const int B = (int)(P.blk_off[k + 1] - a);
            const i64 in = P.in_tok[k];
            const u64 *keys = P.ckeys + a;
            u64 kk0[4];
#pragma unroll
            for (int q = 0; q < 4; q++) kk0[q] = (32 * q + lane < B) ? keys[32 * q + lane] : 0;
            u64 mybits = ~0ULL;
            int myh = 0;
            for (int s0 = 0; s0 < nmine; s0 += 2) {
                const int ns = min(2, nmine - s0);
                Table T2[2];
                bool cand[2];
                int hh[2] = {0, 0};
#pragma unroll
                for (int q = 0; q < 2; q++) {
                    const int gi = base + l0 + s0 + q;
                    cand[q] = q < ns && ((mode != MODE_ENQUEUE) || gi == target);
                    T2[q] = table_of(P, q < ns ? gi : base + l0 + s0);
                }
                if (cand[0] && cand[1]) {
                    u32 m[2][4];
                    probe128<2>(T2, kk0, B, lane, m);
                    hh[0] = lead_hits(m[0]);
                    hh[1] = lead_hits(m[1]);
                } else {
#pragma unroll
                    for (int q = 0; q < 2; q++) if (cand[q]) {
                        u32 m[1][4];
                        probe128<1>(&T2[q], kk0, B, lane, m);
                        hh[q] = lead_hits(m[0]);
                    }
                }
#pragma unroll
                for (int q = 0; q < 2; q++) {
                    if (!cand[q]) continue;
                    if (hh[q] >= 128) hh[q] = B <= 128 ? B : deep_match(T2[q], keys, B, lane);
                    else hh[q] = min(hh[q], B);
                    Inst *sp = st + l0 + s0 + q;
                    const int gi = base + l0 + s0 + q;
                    if (sp->due <= t) {      // snapshot() flushes every candidate (indicators.py:36-65)
                        __syncwarp();
                        if (lane == 0) flush_view(*sp, t);
                        __syncwarp();
                    }
                    const double sc = score_of(P, *sp, hh[q], in);
                    if (P.scores != nullptr && lane == 0) P.scores[gi] = sc;
                    // one 8-B key compare per reference dict lookup + 16 B of view
                    c_bytes += 8ULL * (u64)min(hh[q] + 1, B) + 16ULL;
                    if (lane == s0 + q) { mybits = (u64)__double_as_longlong(sc); myh = hh[q]; }
                }
            }
            if (cta == 0 && warp == 0) c_bytes += 8ULL * (u64)B;   // request chain keys, read once
            const u64 wmin = warp_min_u64(mybits);
            const u32 tmask = __ballot_sync(FULL, lane < nmine && mybits == wmin && wmin != ~0ULL);
            if (lane == 0) { Part q; q.minb = wmin; q.cnt = __popc(tmask); q.err = (u32)werr; wp[par * W + warp] = q; }
            __syncthreads();
            // ---- argmin with the rotating tie-break (policies.py:160-165, 92-101)
            u64 gmin; u32 T; u32 gerr; u32 cincl = 0;
            if (C == 1) {
                Part q; q.minb = ~0ULL; q.cnt = 0; q.err = 0;
                if (lane < W) q = wp[par * W + lane];
                gmin = warp_min_u64(q.minb);
                T = warp_sum(q.minb == gmin ? q.cnt : 0u);
                gerr = __reduce_or_sync(FULL, q.err);
            } else {
                if (warp == 0) {
                    Part q; q.minb = ~0ULL; q.cnt = 0; q.err = 0;
                    if (lane < W) q = wp[par * W + lane];
                    const u64 cmin = warp_min_u64(q.minb);
                    const u32 cc = warp_sum(q.minb == cmin ? q.cnt : 0u);
                    const u32 ce = __reduce_or_sync(FULL, q.err);
                    if (lane < C) {   // push this CTA's partial into every CTA of the cluster (DSMEM)
                        Part *dst = cp + par * C + cta;
                        st_cluster_u64(smem_addr(&dst->minb), (u32)lane, cmin);
                        st_cluster_u64(smem_addr(&dst->cnt), (u32)lane, ((u64)ce << 32) | cc);
                    }
                }
                cluster_sync_all();
                Part q; q.minb = ~0ULL; q.cnt = 0; q.err = 0;
                if (lane < C) q = cp[par * C + lane];
                gmin = warp_min_u64(q.minb);
                const u32 c = (lane < C && q.minb == gmin) ? q.cnt : 0u;
                T = warp_sum(c);
                gerr = __reduce_or_sync(FULL, q.err);
                cincl = warp_incl_scan(c, lane);
            }
            if (gerr) { if (werr == 0) werr = (int)gerr; break; }
            if (T == 0) { werr = 11; break; }                       // NoInstancesError
            u32 kk = 0;
            if (T > 1) {                                            // TieBreaker.pick: tied[counter % len]; counter += 1
                kk = (u32)(counter % (unsigned __int128)T);
                counter += 1;
            }
            int owner_cta = 0;
            u32 kk_local = kk;
            if (C > 1) {                                            // ascending id order = CTA-major
                const u32 ge = __ballot_sync(FULL, lane < C && cincl > kk);
                owner_cta = __ffs(ge) - 1;
                const u32 before = owner_cta > 0 ? __shfl_sync(FULL, cincl, owner_cta - 1) : 0u;
                kk_local = kk - before;
            }
            if (owner_cta == cta) {
                // locate the warp inside this CTA (ascending instance id = warp-major, lane-minor)
                Part q; q.minb = ~0ULL; q.cnt = 0; q.err = 0;
                if (lane < W) q = wp[par * W + lane];
                const u32 c = q.minb == gmin ? q.cnt : 0u;
                const u32 incl = warp_incl_scan(c, lane);
                const u32 ge = __ballot_sync(FULL, lane < W && incl > kk_local);
                const int ow = __ffs(ge) - 1;
                if (warp == ow) {
                    const u32 before = ow > 0 ? __shfl_sync(FULL, incl, ow - 1) : 0u;
                    const int s = nth_set_bit(tmask, (int)(kk_local - before));
                    const int h = __shfl_sync(FULL, myh, s);
                    const int gi = base + l0 + s;
                    commit(P, st + l0 + s, gi, k, h, t, kk0, in, lane, werr);
                    if (P.dec_ns != nullptr && lane == 0) P.dec_ns[k] = (i64)globaltimer();
                }
            }
        }
    }
    // write back
    __syncthreads();
    {
        u64 *dst = (u64 *)(P.inst + base);
        const u64 *src = (const u64 *)st;
        const int words = nloc * (int)(sizeof(Inst) / 8);
        for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
    }
    if (werr && lane == 0) atomicCAS(P.err, 0, werr);
    if (lane == 0 && P.ctr != nullptr) {
        if (c_bytes) atomicAdd(P.ctr + 0, c_bytes);
        if (c_steps) atomicAdd(P.ctr + 1, c_steps);
    }
    if (cta == 0 && threadIdx.x == 0 && mode != MODE_DRAIN) {
        P.tie[0] = (u64)counter;
        P.tie[1] = (u64)(counter >> 64);
    }
    if (C > 1) cluster_sync_all();
}

// ---------------------------------------------------------------- probe batch
// What-if probe: warp per (request, instance) pair against the frozen state.
__global__ void __launch_bounds__(256)
probe_batch_kernel(Params P, i64 r0, i64 nreq, int *out) {
    const i64 wid = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const i64 total = nreq * P.N;
    for (i64 w = wid; w < total; w += ((i64)gridDim.x * blockDim.x) >> 5) {
        const i64 r = r0 + w / P.N;
        const int gi = (int)(w % P.N);
        const i64 a = P.blk_off[r];
        const int B = (int)(P.blk_off[r + 1] - a);
        const int h = warp_probe(table_of(P, gi), P.ckeys + a, B, lane);
        if (lane == 0) out[w] = h;
    }
}

// ---------------------------------------------------------------- cache ops (API)
// op 0: insert_keys(keys, now) -> evicted ; op 1: match_keys(keys) -> hit
__global__ void cache_op_kernel(Params P, int gi, int op, const u64 *keys, int n, i64 now, i64 *result) {
    const int lane = threadIdx.x & 31;
    Table T = table_of(P, gi);
    int werr = 0;
    if (op == 1) {
        int h = warp_probe(T, keys, n, lane);
        if (lane == 0) result[0] = h;
        return;
    }
    Inst *sp = P.inst + gi;
    i64 occ = sp->occ;
    const i64 occ0 = occ;
    occ += warp_unpin_insert(T, keys, n, keys, n, 0, now, lane, werr);
    i64 before_evict = occ;
    if (occ > P.max_occ) werr = DEV_E_TABLE_FULL;
    if (P.cap >= 0 && occ > P.cap && !werr) warp_evict(T, P.cap, occ, lane, werr);
    (void)occ0;
    if (lane == 0) {
        sp->occ = occ;
        result[0] = before_evict - occ;
        if (werr) atomicCAS(P.err, 0, werr);
    }
}
