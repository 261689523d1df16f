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
