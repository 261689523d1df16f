// rsim_route_request's two small kernels around the one-decision replay launch: the request
// comes in as one pinned block (one H2D copy into a device staging buffer) and the decision, the
// per-instance scores and the device error word go out through mapped pinned host memory, so
// one route() call is one copy, three launches and one stream synchronisation (ClusterSim.route,
// cluster.py:130-154).
#pragma once
#include "rsim_device.cuh"

// request block layout (i64 words), written by the host before the launch
enum { RQ_ARRIVAL = 0, RQ_IN, RQ_OUT, RQ_RID, RQ_B, RQ_R0, RQ_NBLK0, RQ_NOUT0, RQ_NO, RQ_NDUP,
       RQ_TRACK, RQ_NEWT, RQ_EXLEN, RQ_CKEY, RQ_HDR = 16 };   // + the detector class (route() with a detector)
// result block layout
enum { RO_CHOSEN = 0, RO_HIT, RO_ERR0, RO_ERR1, RO_ERR2, RO_ERR3, RO_FLAG, RO_HDR = 8 };

// One warp: append the request to the device trace columns (what rsim_load_trace's copies do),
// initialise its result slots, fold its chain keys (one lane: hashing.py:36-47 is sequential)
// and the output-block keys (engine.py:363-372), and install the holders bitmap.
__global__ void __launch_bounds__(32)
route_ingest_kernel(const i64 *__restrict__ rq, i64 *arrival, i64 *in_tok, i64 *out_tok, u64 *rid, i64 *blk_off,
                    i64 *ooff, u64 *blocks, u64 *ckeys, u64 *okeys, int *chosen, int *hit_blocks, i64 *hit_tokens,
                    i64 *first_sched, i64 *first_token, i64 *finish, i64 *route_bs, i64 *dec_ns, u32 *dupmask,
                    int *flag, int *dtid, int *dtw, i64 *dtex, u64 *dtkey) {
    const int lane = threadIdx.x;
    const i64 B = rq[RQ_B], R0 = rq[RQ_R0], nb0 = rq[RQ_NBLK0], no0 = rq[RQ_NOUT0], no = rq[RQ_NO];
    const i64 ndup = rq[RQ_NDUP];
    const i64 *src = rq + RQ_HDR + ndup;
    for (i64 j = lane; j < B; j += 32) blocks[nb0 + j] = (u64)src[j];
    for (i64 j = lane; j < ndup; j += 32) dupmask[j] = (u32)rq[RQ_HDR + j];
    if (lane == 0) {
        arrival[R0] = rq[RQ_ARRIVAL]; in_tok[R0] = rq[RQ_IN]; out_tok[R0] = rq[RQ_OUT]; rid[R0] = (u64)rq[RQ_RID];
        blk_off[R0] = nb0; blk_off[R0 + 1] = nb0 + B;
        ooff[R0] = no0; ooff[R0 + 1] = no0 + no;
        chosen[R0] = -1; hit_blocks[R0] = 0;
        hit_tokens[R0] = first_sched[R0] = first_token[R0] = finish[R0] = route_bs[R0] = dec_ns[R0] = -1;
        if (dtid != nullptr) {                 // the request's detector track; a new track's exemplar is
            dtid[R0] = (int)rq[RQ_TRACK];      // this request's own leading chain keys
            const i64 t = rq[RQ_NEWT];
            if (t >= 0) { dtw[t] = (int)rq[RQ_EXLEN]; dtex[t] = nb0; dtkey[t] = (u64)rq[RQ_CKEY]; }
        }
    }
    __syncwarp();
    if (lane == 0) {
        bool bad = false;
        u64 acc = RSIM_GOLDEN;
#pragma unroll 4
        for (i64 j = 0; j < B; j++) {
            acc = combine64(acc, (u64)src[j]);
            bad |= (acc == 0ULL);
            ckeys[nb0 + j] = acc;
        }
        const u64 salt = combine64(combine64(RSIM_GOLDEN, RSIM_OUTPUT_SALT), (u64)rq[RQ_RID]);
        for (i64 i = 0; i < no; i++) {
            acc = combine64(acc, combine64(salt, (u64)i));
            bad |= (acc == 0ULL);
            okeys[no0 + i] = acc;
        }
        *flag = bad ? 1 : 0;
    }
}

__global__ void route_out_kernel(const int *__restrict__ chosen, const i64 *__restrict__ hit_tokens, i64 r,
                                 const double *__restrict__ scores, int nscores, const int *__restrict__ err,
                                 const int *__restrict__ flag, i64 *ro) {
    const int t = threadIdx.x;
    if (t == 0) {
        ro[RO_CHOSEN] = chosen[r]; ro[RO_HIT] = hit_tokens[r];
        ro[RO_ERR0] = err[0]; ro[RO_ERR1] = err[1]; ro[RO_ERR2] = err[2]; ro[RO_ERR3] = err[3];
        ro[RO_FLAG] = *flag;
    }
    for (int i = t; i < nscores; i += blockDim.x) ro[RO_HDR + i] = __double_as_longlong(scores[i]);
}

// ---- route(): the whole call in ONE launch (plain policies, no staleness / detector, one rank,
// N <= 1024 instances): one CTA of NW = ceil(N / 32) warps, each owning <= 32 instances of the
// shard. Warp 0 ingests the request (as route_ingest_kernel) and stages it; every warp probes
// and scores its instances against the live state in global memory (the replay kernel's
// probe_hits / probe_hits_sparse / score_phase on global Inst records); the block reduces the
// (score, tie count) partials in instance order, applies the TieBreaker counter
// (cluster.py:90-94), and the owning warp enqueues (commit + the touch / pin of the hit chain,
// engine.py:262-289). Results go straight to mapped pinned memory (route_out_kernel's layout).
#define RK_MAXW 32
__global__ void __launch_bounds__(32 * RK_MAXW, 1)
route_kernel(const __grid_constant__ Params P, const i64 *__restrict__ rq, i64 *ro, int nsc, u64 *blocks) {
    extern __shared__ __align__(16) unsigned char rk_smem[];
    __shared__ ReqStage R;
    __shared__ u64 pmin[RK_MAXW];
    __shared__ u32 pcnt[RK_MAXW];
    __shared__ int dec_owner, dec_kk, dec_err;
    WarpBuf *wbuf = reinterpret_cast<WarpBuf *>(rk_smem);
    Inst *st = reinterpret_cast<Inst *>(wbuf + (blockDim.x >> 5));   // the shard's instance records
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, NW = blockDim.x >> 5;
    WarpBuf &WB = wbuf[warp];
    const i64 B = rq[RQ_B], R0 = rq[RQ_R0], nb0 = rq[RQ_NBLK0], no0 = rq[RQ_NOUT0], no = rq[RQ_NO];
#ifdef RSIM_ROUTE_TIMING
    if (threadIdx.x == 0) ro[RO_HDR + nsc + 0] = (i64)globaltimer();
#endif
    const i64 ndup = rq[RQ_NDUP];
    const i64 *src = rq + RQ_HDR + ndup;
    if (warp == 0) {                                   // ingest (route_ingest_kernel's body)
        for (i64 j = lane; j < B; j += 32) blocks[nb0 + j] = (u64)src[j];
        if (lane == 0) {
            const_cast<i64 *>(P.arrival)[R0] = rq[RQ_ARRIVAL]; const_cast<i64 *>(P.in_tok)[R0] = rq[RQ_IN]; const_cast<i64 *>(P.out_tok)[R0] = rq[RQ_OUT];
            const_cast<u64 *>(P.rid)[R0] = (u64)rq[RQ_RID];
            const_cast<i64 *>(P.blk_off)[R0] = nb0; const_cast<i64 *>(P.blk_off)[R0 + 1] = nb0 + B;
            const_cast<i64 *>(P.ooff)[R0] = no0; const_cast<i64 *>(P.ooff)[R0 + 1] = no0 + no;
            P.chosen[R0] = -1; P.hit_blocks[R0] = 0;
            P.hit_tokens[R0] = P.first_sched[R0] = P.first_token[R0] = P.finish[R0] = P.route_bs[R0] = -1;
            if (P.dec_ns != nullptr) P.dec_ns[R0] = -1;
            bool bad = false;
            u64 acc = RSIM_GOLDEN;
#pragma unroll 4
            for (i64 j = 0; j < B; j++) {
                acc = combine64(acc, (u64)src[j]);
                bad |= (acc == 0ULL);
                const_cast<u64 *>(P.ckeys)[nb0 + j] = acc;
                if (j < 128) { R.keys[j] = acc; R.home[j] = tab_home(acc, P.slog2); }
            }
            const u64 salt = combine64(combine64(RSIM_GOLDEN, RSIM_OUTPUT_SALT), (u64)rq[RQ_RID]);
            for (i64 i = 0; i < no; i++) {
                acc = combine64(acc, combine64(salt, (u64)i));
                bad |= (acc == 0ULL);
                const_cast<u64 *>(P.okeys)[no0 + i] = acc;
            }
            R.t = rq[RQ_ARRIVAL]; R.a = nb0; R.in = rq[RQ_IN]; R.oa = no0; R.B = (int)B; R.out = (int)rq[RQ_OUT];
            ro[RO_FLAG] = bad ? 1 : 0;
        }
    }
    if (lane == 0) {
        WB.c_bytes = 0; WB.c_steps = 0; WB.werr = 0; WB.fins = 0; WB.spk = -1;
        WB.fin.dnf = 0; WB.fin.npark = 0; WB.fin.tpn = 0; WB.fin.lnext = WB.fin.lend = 0;
    }
#ifdef RSIM_ROUTE_TIMING
    if (threadIdx.x == 0) ro[RO_HDR + nsc + 1] = (i64)globaltimer();
#endif
    {   // the instance records into shared memory (one coalesced pass; the snapshot flushes and the
        // commit's read-modify-writes then cost shared-memory latency), back at the end
        const u64 *src = reinterpret_cast<const u64 *>(P.inst);
        u64 *dst = reinterpret_cast<u64 *>(st);
        const int words = P.N * (int)(sizeof(Inst) / 8);
        for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
#ifdef RSIM_ROUTE_TIMING
    if (threadIdx.x == 0) ro[RO_HDR + nsc + 2] = (i64)globaltimer();
#endif
    // probe + score this warp's instances
    const int ipw = (P.N + NW - 1) / NW, l0 = warp * ipw;
    const int n = max(0, min(ipw, P.N - l0));
    u64 mybits = ~0ULL;
    u32 tmask = 0u;
    if (n > 0) {
        if (n >= 2 && R.B <= 128) probe_hits_sparse(P, 0, l0, n, R, MODE_ROUTE, -1, 0u, lane, WB.hit);
        else probe_hits(P, 0, l0, n, R, MODE_ROUTE, -1, 0u, lane, WB.hit, WB.slot[0]);
        u64 bits_bs;
        mybits = score_phase(P, st, 0, l0, n, R, MODE_ROUTE, -1, lane, WB, bits_bs, false, P.bsn, false, nullptr);
    }
#ifdef RSIM_ROUTE_TIMING
    if (threadIdx.x == 0) ro[RO_HDR + nsc + 3] = (i64)globaltimer();
#endif
    const u64 wmin = warp_min_u64(lane < n ? mybits : ~0ULL);
    tmask = __ballot_sync(FULL, lane < n && mybits == wmin && wmin != ~0ULL);
    if (lane == 0) { pmin[warp] = wmin; pcnt[warp] = (u32)__popc(tmask); }
    __syncthreads();
#ifdef RSIM_ROUTE_TIMING
    if (threadIdx.x == 0) ro[RO_HDR + nsc + 4] = (i64)globaltimer();
#endif
    if (warp == 0) {                                   // argmin over the warps in instance order + tie-break
        const u64 m = lane < NW ? pmin[lane] : ~0ULL;
        const u64 g = warp_min_u64(m);
        const u32 c = (lane < NW && m == g && g != ~0ULL) ? pcnt[lane] : 0u;
        const u32 T = __reduce_add_sync(FULL, c);
        u32 kk = 0;
        if (T > 1) {                                   // TieBreaker.pick: tied[counter % len]; counter += 1
            const u64 lo = P.tie[0], hi = P.tie[1];
            kk = mod_counter(lo, hi, T);
            __syncwarp();
            if (lane == 0) { P.tie[0] = lo + 1; P.tie[1] = hi + (lo + 1 < lo); }
        }
        const u32 incl = warp_incl_scan(c, lane);
        const u32 ge = __ballot_sync(FULL, c > 0 && incl > kk);
        const int ow = T ? __ffs(ge) - 1 : -1;
        const u32 bef = ow > 0 ? __shfl_sync(FULL, incl, ow - 1) : 0u;
        if (lane == 0) { dec_owner = ow; dec_kk = (int)(kk - bef); dec_err = T ? 0 : 11; }   // 11: NoInstancesError
    }
    __syncthreads();
#ifdef RSIM_ROUTE_TIMING
    if (threadIdx.x == 0) ro[RO_HDR + nsc + 5] = (i64)globaltimer();
#endif
    if (warp == dec_owner) {
        const int s = nth_set_bit_warp(tmask, dec_kk, lane);
        const int gi = l0 + s, gch = P.gbase + gi;
        const int h = WB.hit[s];
        int werr = 0;
        if (ndup > 0 && ((rq[RQ_HDR + (gch >> 5)] >> (gch & 31)) & 1)) {   // holders bitmap of this call
            werr = DEV_E_DUPLICATE;                    // chosen (the counter moved), never enqueued
        } else {
            commit(P, st + gi, gi, R0, h, R.t, R.keys, nullptr, R.a, R.B, R.in, R.out, R.oa, lane, werr, WB.fin, false);
            flush_touch_pin(P, WB.fin, lane, &werr);
        }
        if (lane == 0 && werr) atomicCAS(P.err, 0, werr);
    }
#ifdef RSIM_ROUTE_TIMING
    if (threadIdx.x == 0) ro[RO_HDR + nsc + 6] = (i64)globaltimer();
#endif
    if (lane == 0 && WB.werr) atomicCAS(P.err, 0, WB.werr);
    if (dec_err && threadIdx.x == 0) atomicCAS(P.err, 0, dec_err);
    __syncthreads();
    {
        u64 *dst = reinterpret_cast<u64 *>(P.inst);
        const u64 *src = reinterpret_cast<const u64 *>(st);
        const int words = P.N * (int)(sizeof(Inst) / 8);
        for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
    }
#ifdef RSIM_ROUTE_TIMING
    if (threadIdx.x == 0) ro[RO_HDR + nsc + 7] = (i64)globaltimer();
#endif
    __threadfence();
    if (threadIdx.x == 0) {
        ro[RO_CHOSEN] = P.chosen[R0]; ro[RO_HIT] = P.hit_tokens[R0];
        ro[RO_ERR0] = P.err[0]; ro[RO_ERR1] = P.err[1]; ro[RO_ERR2] = P.err[2]; ro[RO_ERR3] = P.err[3];
    }
    for (int i = threadIdx.x; i < nsc; i += blockDim.x) ro[RO_HDR + i] = __double_as_longlong(P.scores[i]);
}
