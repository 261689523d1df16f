// rsim_detector.cuh -- the prefix-hotspot detector (reference detector.py:164-377) on
// the replay kernel's control warp.
//
// A class is the set of requests sharing their leading class_key_blocks blocks; the
// host numbers classes densely by first arrival (tracks). Every CTA's control warp runs
// the same state machine on its own copy (deterministic inputs); CTA 0's copy emits the
// rows and is written back. Per decision k:
//   * instance warps score three argmin branches -- the policy's score, the same with
//     the holders of class(k) (instances holding its first w_k chain keys, i.e. hit
//     blocks >= w_k) excluded, and least batch size -- plus the holder count and the
//     min / sum of the holder-free products p_tokens * max(bs, 1) (detector.py:310-316);
//     they also count the holders of the few tracks the control warp listed for k
//     (alarmed classes and, when a window closes, the rows' classes);
//   * the control warp picks the branch from verdict(k) (detector.py:281-289; fail open,
//     policies.py:229-236), then runs observe(k) (detector.py:292-330) before releasing
//     the decision, and prepares verdict(k+1) and the holder list of k+1.
// State lives in global memory and is touched only by the control warp. Times are
// integers in us; the float arithmetic follows CPython's (correctly rounded IEEE).
#pragma once
#include "rsim_cache.cuh"

#define RSIM_DLMAX 64                  // tracks re-evaluated in one decision
#define RSIM_DET_SMEM_T 512            // tracks kept in shared memory during a replay (more: global)
enum { DG_TOTAL = 0, DG_WIDX, DG_HASW, DG_FIRSTV, DG_NROWS, DG_TOTH, DG_TOTN, DG_HZ, DG_NTR, DG_TTSEC, DG_TTCNT,
       DG_N };

struct DTrack {                        // _Track (detector.py:151-161)
    i64 wc, wh, streak, last_sus;      // window_count, window_hit_tokens, streak, last_suspect_us
    i64 tsec, tcnt, thits;             // the newest bucket (entry bn - 1; older ones in the global ring)
    int bh, bn;                        // bucket deque [bh, bn)
    int flags;                         // bit0 suspect_now, bit1 alarmed
    int pad;
};

// where the control warp keeps the detector state: shared memory for a replay (copied in
// at launch, out at exit), global memory for the finalize kernel or very many classes
struct DetView {
    DTrack *tr; const u64 *key; i64 *g;
    i64 *bk, *tot;                     // this CTA's global bucket rings (older buckets)
    bool rows;                         // this copy emits the DetectorRows (CTA 0)
};

struct DetCtl {                        // control warp -> instance warps, decision k
    u64 mbd[2];                        // [parity] the instance warps counted the listed holders
    i64 list_seq;                      // (decision << 8) | nl: the list below belongs to that decision
    i64 pad_;
    u64 own[2][2];                     // [parity] (hit blocks, product) of the chosen instance, sent by its warp
    int verdict, w, nl, nrow;          // 0 none / 1 exclude holders / 2 force least_bs; w_k; |lst|; rows
    int lst[RSIM_DLMAX];               // tracks whose holders the instance warps count
    u32 cnt[RSIM_DLMAX];               // holder counts of lst, summed over the cluster's warps
    i64 g[DG_N + 1];                   // detector scalars while the replay runs
};
static_assert(sizeof(DetCtl) % 16 == 0 && offsetof(DetCtl, own) % 16 == 0, "st.async targets are 16-B aligned");

__device__ __forceinline__ bool det_rank_before(const DTrack &a, u64 ka, const DTrack &b, u64 kb) {
    if (a.wh != b.wh) return a.wh > b.wh;          // sorted by (-hits, -count, key), detector.py:210-213
    if (a.wc != b.wc) return a.wc > b.wc;
    return ka < kb;
}

// tracks ranked ahead of t among the created ones (warp-wide)
__device__ int det_ahead(const DetView &V, int ntr, int t, int lane) {
    const i64 wh = V.tr[t].wh, wc = V.tr[t].wc;
    const u64 km = V.key[t];
    int c = 0;
    for (int j = lane; j < ntr; j += 32) {
        const i64 h = V.tr[j].wh, w = V.tr[j].wc;
        c += (j != t) && (h != wh ? h > wh : (w != wc ? w > wc : V.key[j] < km));
    }
    return warp_sum(c);
}
__device__ __forceinline__ bool det_in_top(const Params &P, const DetView &V, int ntr, int t, int lane) {   // _top_keys
    return ntr <= P.dtopk || det_ahead(V, ntr, t, lane) < P.dtopk;
}

__device__ __forceinline__ bool phase1_suspect(double x, i64 nh, i64 no) {   // detector.py:85-101
    if (x <= 0.0 || nh == 0) return false;
    const double rem = __dsub_rn(1.0, x);
    if (rem <= 0.0 || no == 0) return true;
    return __ddiv_rn(x, rem) > __ddiv_rn((double)nh, (double)no);
}

__device__ __forceinline__ double det_fraction(const DetView &V, const DTrack &t) {
    const i64 tot = V.g[DG_TOTAL];
    return tot ? __ddiv_rn((double)t.wc, (double)tot) : 0.0;
}

// _evaluate_phase1 (detector.py:225-245), lane 0
__device__ bool det_phase1(const Params &P, const DetView &V, int t, i64 nh, i64 now) {
    DTrack &tr = V.tr[t];
    const bool sus = phase1_suspect(det_fraction(V, tr), nh, (i64)P.N - nh);
    tr.flags = (tr.flags & ~1) | (sus ? 1 : 0);
    if (sus) {
        tr.last_sus = now;
        if (V.g[DG_FIRSTV] < 0) V.g[DG_FIRSTV] = now;
    } else {
        tr.streak = 0;
    }
    if ((tr.flags & 2) && !sus && now - tr.last_sus >= P.dcool) { tr.flags &= ~2; tr.streak = 0; }
    return sus;
}

// CPython float floor division (floatobject.c float_floor_div)
__device__ __forceinline__ double py_floordiv(double a, double b) {
    const double mod = fmod(a, b);
    double div = __ddiv_rn(__dsub_rn(a, mod), b);
    if (mod != 0.0 && ((b < 0) != (mod < 0))) div = __dsub_rn(div, 1.0);
    if (div != 0.0) {
        double fl = floor(div);
        if (__dsub_rn(div, fl) > 0.5) fl = __dadd_rn(fl, 1.0);
        return fl;
    }
    return copysign(0.0, __ddiv_rn(a, b));
}
__device__ __forceinline__ i64 det_window_of(const Params &P, i64 now) {   // _roll_window index
    return (i64)py_floordiv(__ddiv_rn((double)now, 1e6), P.dwin);
}

// does a window close at `now` (_roll_window's idx > _window_idx)? The exact CPython index
// (fmod-based, slow on the GPU) only within a few us of the boundary; elsewhere the answer
// is certain (the float error is ~1e-4 us at 1e12 us).
__device__ __forceinline__ bool det_rolls(const Params &P, const i64 *g, i64 now) {
    const double tb = __dmul_rn(__dmul_rn((double)(g[DG_WIDX] + 1), P.dwin), 1e6);
    if ((double)now < tb - 4.0) return false;
    if ((double)now > tb + 4.0) return true;
    return det_window_of(P, now) > g[DG_WIDX];
}

// one DetectorRow (detector.py:356-370), lane 0
__device__ void det_emit_row(const Params &P, const DetView &V, int t, i64 widx, i64 nh) {
    const i64 n = V.g[DG_NROWS];
    if (V.rows && n < P.drows_cap) {
        const DTrack &tr = V.tr[t];
        i64 *r = P.drows + 7 * n;
        r[0] = __double_as_longlong(__dmul_rn((double)widx, P.dwin));
        r[1] = (i64)V.key[t];
        r[2] = __double_as_longlong(det_fraction(V, tr));
        r[3] = nh; r[4] = (i64)P.N - nh;
        r[5] = tr.flags & 1;
        r[6] = (tr.flags & 2) ? 2 : (tr.flags & 1);
    }
    V.g[DG_NROWS] = n + 1;
}

// the top tracks in class-key order (_emit_rows' sorted(_top_keys())) -> out[], returns count (warp-wide)
__device__ int det_top_sorted(const Params &P, const DetView &V, int *out, int cap, int lane) {
    const int ntr = (int)V.g[DG_NTR];
    int m = 0;
    for (int t = 0; t < ntr; t++) {
        if (!det_in_top(P, V, ntr, t, lane)) continue;
        if (lane == 0) {
            if (m >= cap) { atomicCAS(P.err, 0, DEV_E_DETECTOR); }
            else {
                int j = m;                                  // insertion by class key
                while (j > 0 && V.key[out[j - 1]] > V.key[t]) { out[j] = out[j - 1]; j--; }
                out[j] = t;
            }
        }
        m++;
    }
    __syncwarp();
    return min(m, cap);
}

// verdict(k) and the holder list of decision k (before its partials), control warp
__device__ void det_prepare(const Params &P, const DetView &V, DetCtl &D, i64 now, int tid, int w, int lane) {
    const int ntr = (int)V.g[DG_NTR];
    int nrow = 0;
    if (V.g[DG_HASW] && det_rolls(P, V.g, now))             // a window closes at observe(k)
        nrow = det_top_sorted(P, V, D.lst, RSIM_DLMAX, lane);
    int nl = nrow;
    for (int t0 = 0; t0 < ntr; t0 += 32) {                  // alarmed classes decay at observe(k)
        const int t = t0 + lane;
        const u32 al = __ballot_sync(FULL, t < ntr && (V.tr[t].flags & 2));
        const int pos = nl + __popc(al & lanemask_lt());
        if ((al >> lane) & 1u) { if (pos < RSIM_DLMAX) D.lst[pos] = t; else atomicCAS(P.err, 0, DEV_E_DETECTOR); }
        nl += __popc(al);
    }
    if (lane == 0) {
        D.nrow = nrow; D.nl = min(nl, RSIM_DLMAX);
        D.w = w;
        D.verdict = (tid < ntr && (V.tr[tid].flags & 2)) ? (P.dforce ? 2 : 1) : 0;
    }
    __syncwarp();
}

// Detector.observe (detector.py:292-330) for decision k, control warp. nh: holders of
// class(k); pmin / psum: min / sum of holder-free products; cnt: holder counts of D.lst.
__device__ void det_observe(const Params &P, const DetView &V, DetCtl &D, int tid, i64 now, int lane, i64 hit_tok,
                            bool chosen_held, i64 prod_c, i64 nh, u64 pmin, i64 psum, const u32 *cnt) {
    i64 *g = V.g;
    // _roll_window (detector.py:340-348)
    if (!g[DG_HASW]) {
        if (lane == 0) { g[DG_WIDX] = det_window_of(P, now); g[DG_HASW] = 1; }
    } else if (det_rolls(P, g, now)) {
        if (lane == 0) {
            for (int j = 0; j < D.nrow; j++) det_emit_row(P, V, D.lst[j], g[DG_WIDX], (i64)cnt[j]);
            g[DG_WIDX] = det_window_of(P, now);
        }
    }
    __syncwarp();
    // _expire (detector.py:177-185): only when the horizon moved -- or, for windows under one
    // second (int(window_s) == 0), always: the last bump's bucket is then already at the horizon
    const i64 horizon = now / 1000000 - P.dwin_i;
    const int BC = 1 << P.dbclog2, bm = BC - 1;
    int ntr = (int)g[DG_NTR];
    if (horizon > g[DG_HZ] || P.dwin_i == 0) {
        for (int t = lane; t < ntr; t += 32) {
            DTrack &tr = V.tr[t];
            const i64 *b = V.bk + (size_t)t * BC * 3;
            while (tr.bn > tr.bh) {
                const bool tail = tr.bh == tr.bn - 1;
                const i64 sec = tail ? tr.tsec : b[(tr.bh & bm) * 3];
                if (sec > horizon) break;
                tr.wc -= tail ? tr.tcnt : b[(tr.bh & bm) * 3 + 1];
                tr.wh -= tail ? tr.thits : b[(tr.bh & bm) * 3 + 2];
                tr.bh++;
            }
        }
        if (lane == 0) {
            i64 h = g[DG_TOTH];
            const i64 n = g[DG_TOTN];
            while (n > h) {
                const bool tail = h == n - 1;
                if ((tail ? g[DG_TTSEC] : V.tot[(h & bm) * 2]) > horizon) break;
                g[DG_TOTAL] -= tail ? g[DG_TTCNT] : V.tot[(h & bm) * 2 + 1];
                h++;
            }
            g[DG_TOTH] = h;
            g[DG_HZ] = horizon;
        }
    }
    __syncwarp();
    // new track (classes are numbered by first arrival) + _bump (detector.py:187-203); the
    // newest bucket stays in the track, older ones go to the global ring
    if (lane == 0) {
        if (tid == ntr) { g[DG_NTR] = ntr + 1; V.tr[tid].last_sus = -1; }
        const i64 sec = now / 1000000;
        const i64 h = g[DG_TOTH], n = g[DG_TOTN];
        if (n > h && g[DG_TTSEC] == sec) g[DG_TTCNT] += 1;
        else if (n - h >= BC) atomicCAS(P.err, 0, DEV_E_DETECTOR);
        else {
            if (n > h) { V.tot[((n - 1) & bm) * 2] = g[DG_TTSEC]; V.tot[((n - 1) & bm) * 2 + 1] = g[DG_TTCNT]; }
            g[DG_TTSEC] = sec; g[DG_TTCNT] = 1; g[DG_TOTN] = n + 1;
        }
        g[DG_TOTAL] += 1;
        DTrack &tr = V.tr[tid];
        if (tr.bn > tr.bh && tr.tsec == sec) { tr.tcnt += 1; tr.thits += hit_tok; }
        else if (tr.bn - tr.bh >= BC) atomicCAS(P.err, 0, DEV_E_DETECTOR);
        else {
            if (tr.bn > tr.bh) {
                i64 *b = V.bk + (size_t)tid * BC * 3 + ((tr.bn - 1) & bm) * 3;
                b[0] = tr.tsec; b[1] = tr.tcnt; b[2] = tr.thits;
            }
            tr.tsec = sec; tr.tcnt = 1; tr.thits = hit_tok; tr.bn++;
        }
        tr.wc += 1; tr.wh += hit_tok;
    }
    __syncwarp();
    ntr = (int)g[DG_NTR];
    // hotspot candidates: classes enjoying hits, among the top ones
    if (V.tr[tid].wh > 0 && det_in_top(P, V, ntr, tid, lane) && lane == 0) {
        if (det_phase1(P, V, tid, nh, now)) {               // _evaluate_phase2 (detector.py:247-270)
            DTrack &tr = V.tr[tid];
            const i64 no = (i64)P.N - nh;                   // decision.filtered is a subset of the holders
            bool q = false;
            if (chosen_held && no > 0) {
                const double ref = P.dmean ? __ddiv_rn((double)psum, (double)no) : (double)(i64)pmin;
                q = (double)prod_c <= ref;
            }
            tr.streak = q ? tr.streak + 1 : 0;
            if ((double)tr.streak > __dmul_rn(P.dmult, (double)nh)) { tr.flags |= 2; tr.last_sus = now; }
        }
    }
    __syncwarp();
    if (lane == 0)                                          // alarmed classes decay toward benign
        for (int j = D.nrow; j < D.nl; j++) {
            const int t = D.lst[j];
            if (t != tid && (V.tr[t].flags & 2)) det_phase1(P, V, t, (i64)cnt[j], now);
        }
    __syncwarp();
}

// holders of track t among instances [gi0, gi0 + n): lane s checks instance gi0 + s
__device__ __forceinline__ bool det_holds(const Params &P, int t, int gi) {
    const Table T = table_of(P, gi);
    const u64 *ex = P.ckeys + P.dtex[t];
    const int w = P.dtw[t];
    for (int j = 0; j < w; j++) if (tab_find(T, ex[j]) < 0) return false;
    return true;
}

// Detector.finalize (detector.py:373-377): the last window's rows on the final tables
__global__ void det_finalize_kernel(const Params P) {
    __shared__ int lst[RSIM_DLMAX];
    const int lane = threadIdx.x;
    const DetView V{P.dtr, P.dtkey, P.dglob, P.dbk, P.dtot, true};
    if (!P.dglob[DG_HASW] || P.dglob[DG_NTR] == 0) return;
    const int m = det_top_sorted(P, V, lst, RSIM_DLMAX, lane);
    for (int j = 0; j < m; j++) {
        int c = 0;
        for (int gi = lane; gi < P.N; gi += 32) c += det_holds(P, lst[j], gi);
        c = warp_sum(c);
        if (lane == 0) det_emit_row(P, V, lst[j], P.dglob[DG_WIDX], c);
        __syncwarp();
    }
}
