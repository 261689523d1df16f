// rsim_synth.cuh -- device generate_synthetic (reference trace.py:218-268).
//
// The reference draws from Python's random.Random (CPython _randommodule.c: MT19937 seeded
// by init_by_array over the 32-bit words of abs(seed)) in a fixed order:
//   per class ci, stream A = Random(stable_key(seed, 0x5EED0003, ci)): arrival gaps
//     expovariate(weight * mean_rate) = -log(1 - random()) / rate, t0 = gap, t += gap while
//     t < duration (trace.py:228-237; random() = ((w0 >> 5) * 2^26 + (w1 >> 6)) * 2^-53);
//   arrivals sorted as (t, ci, seq) tuples (trace.py:238);
//   per class, stream B = Random(stable_key(seed, 0x5EED0003, ci, 1)): for each of its
//     requests in arrival order randint(*suffix_blocks) then randint(*output_tokens)
//     (trace.py:243-252; randint = lo + _randbelow(hi - lo + 1), _randbelow = getrandbits(k)
//     = w >> (32 - k), k = bit_length(n), redrawn while >= n);
//   blocks = shared chain stable_key(seed, 0x5EED0001, ci, pos) then fresh suffix
//     stable_key(seed, 0x5EED0002, ci, seq, pos); class_key = stable_key(0xC1A55000, b0[, b1]).
// Every value is integer arithmetic or a correctly specified IEEE operation except log, which
// is glibc's (rsim_log.h), so the device trace is bit-identical to the reference's.
//
// Kernels (streams are sequential per class, everything after is data-parallel):
//   synth_arrivals_kernel  one warp per class: the warp twists MT19937 624 words at a time,
//                          lanes turn word pairs into gaps (glibc_log), lane 0 folds the
//                          gaps in order (the float sum is sequential by definition)
//   synth_sizes_kernel     one warp per class: the rejection sampler over the class's stream,
//                          32 words per step by a scan of its two-state machine
//   synth_order_kernel     thread per arrival: rank in the (t, ci, seq) order by binary
//                          search in the other classes' sorted times; scatters the rows
//   (cub inclusive scan of block counts -> blk_off)
//   synth_blocks_kernel    warp per request: block hashes (coalesced), class_key, tokens
#pragma once
#include "rsim_device.cuh"
#include "rsim_log.h"

#define SYN_SHARED_SALT 0x5EED0001ULL
#define SYN_SUFFIX_SALT 0x5EED0002ULL
#define SYN_RNG_SALT 0x5EED0003ULL
#define SYN_CLASS_SALT 0xC1A55000ULL
#define MT_N 624
#define MT_M 397

struct SynClass {           // one rsim_synth_class, device copy
    double rate;            // weight * mean_rate_rps (trace.py:230)
    long long shared, suf_lo, suf_hi, out_lo, out_hi;
};

__device__ const double g_log_tab[256] = RSIM_LOG_TAB_INIT;

// init_by_array(key = 32-bit words of the 64-bit seed, little end first; one word if < 2^32)
__device__ void mt_seed(u32 *mt, u64 seed) {
    u32 key[2] = {(u32)seed, (u32)(seed >> 32)};
    const int klen = (seed >> 32) ? 2 : 1;
    mt[0] = 19650218u;
    for (int i = 1; i < MT_N; i++) mt[i] = 1812433253u * (mt[i - 1] ^ (mt[i - 1] >> 30)) + (u32)i;
    int i = 1, j = 0;
    for (int k = MT_N; k; k--) {
        mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1664525u)) + key[j] + (u32)j;
        i++; j++;
        if (i >= MT_N) { mt[0] = mt[MT_N - 1]; i = 1; }
        if (j >= klen) j = 0;
    }
    for (int k = MT_N - 1; k; k--) {
        mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1566083941u)) - (u32)i;
        i++;
        if (i >= MT_N) { mt[0] = mt[MT_N - 1]; i = 1; }
    }
    mt[0] = 0x80000000u;
}

// The 624-word regeneration by one warp in 32-word chunks, in order: mt[k] reads mt[k+1]
// (old: read before the chunk writes) and mt[k+397 mod 624] (old for k < 227, already new
// for k >= 227 -- an earlier chunk), exactly the sequential recurrence.
__device__ __forceinline__ void mt_twist(u32 *mt, int lane) {
    for (int base = 0; base < MT_N; base += 32) {
        const int k = base + lane;
        u32 nv = 0;
        if (k < MT_N) {
            const u32 y = (mt[k] & 0x80000000u) | (mt[k + 1 < MT_N ? k + 1 : 0] & 0x7fffffffu);
            nv = mt[k + MT_M < MT_N ? k + MT_M : k + MT_M - MT_N] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
        }
        __syncwarp();
        if (k < MT_N) mt[k] = nv;
        __syncwarp();
    }
}

__device__ __forceinline__ u32 mt_temper(u32 y) {
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    return y ^ (y >> 18);
}

__device__ __forceinline__ u64 syn_key(u64 acc, u64 v) { return combine64(acc, v); }

// times[toff[c] ..] gets class c's arrival times (at most cap = toff[c+1]-toff[c] written);
// count[c] = the true number (a count above cap asks the host to rerun with more room).
__global__ void __launch_bounds__(32)
synth_arrivals_kernel(const SynClass *__restrict__ cls, u64 seed, double duration,
                      const i64 *__restrict__ toff, double *__restrict__ times, i64 *__restrict__ count) {
    __shared__ u32 mt[MT_N];
    __shared__ double gap[MT_N / 2], tsum[MT_N / 2];
    const int c = blockIdx.x, lane = threadIdx.x;
    if (lane == 0) mt_seed(mt, syn_key(syn_key(syn_key(RSIM_GOLDEN, seed), SYN_RNG_SALT), (u64)c));
    __syncwarp();
    const double rate = cls[c].rate;
    const i64 cap = toff[c + 1] - toff[c];
    double *out = times + toff[c];
    double t = 0.0;
    i64 n = 0;
    bool first = true, done = false;
    while (!done) {
        mt_twist(mt, lane);
        for (int j = lane; j < MT_N / 2; j += 32) {
            const u32 a = mt_temper(mt[2 * j]) >> 5, b = mt_temper(mt[2 * j + 1]) >> 6;
            const double u = __dmul_rn(__dadd_rn(__dmul_rn((double)a, 67108864.0), (double)b),
                                       1.0 / 9007199254740992.0);
            gap[j] = __ddiv_rn(-glibc_log(__dsub_rn(1.0, u), g_log_tab), rate);
        }
        __syncwarp();
        if (lane == 0) {                 // the float sum is sequential by definition: lane 0
            int j0 = 0;                  // runs only the add chain (loads are independent of t)
            if (first) { t = gap[0]; tsum[0] = t; j0 = 1; first = false; }
            #pragma unroll 8
            for (int j = j0; j < MT_N / 2; j++) { t = __dadd_rn(t, gap[j]); tsum[j] = t; }
        }
        __syncwarp();
        for (int base = 0; base < MT_N / 2; base += 32) {   // keep the prefix below duration
            const int j = base + lane;
            const bool in = j < MT_N / 2;
            const u32 bad = __ballot_sync(FULL, in && !(tsum[in ? j : 0] < duration));
            const int m = bad ? __ffs(bad) - 1 : min(32, MT_N / 2 - base);   // valid: [0, m)
            if (lane < m && n + lane < cap) out[n + lane] = tsum[j];
            n += m;
            if (bad) { done = true; break; }
        }
        done = __shfl_sync(FULL, done, 0);
    }
    if (lane == 0) count[c] = n;
}

// Bits a 64-bit (hi - lo + 1) needs; ranges wider than 2^32 are refused by the host.
__device__ __forceinline__ int syn_bitlen(u64 n) { return 64 - __clzll((long long)n); }

// nsuf / nout[coff[c] + seq]: the class's size draws in seq (= arrival) order; coff is the
// exclusive prefix of the classes' arrival counts. The sampler is a two-state machine over the
// stream's words (state 0: the suffix draw of the next request, 1: its output draw; a word
// below the state's bound is accepted and flips the state, one above is redrawn). Each word is
// a map {0,1} -> {0,1}; maps compose associatively, so a warp takes 32 words at once: a
// shuffle scan of the maps gives every lane its entry state, a ballot numbers the accepted
// draws, and accepted lanes write their draw in parallel.
__global__ void __launch_bounds__(32)
synth_sizes_kernel(const SynClass *__restrict__ cls, u64 seed, const i64 *__restrict__ coff,
                   int *__restrict__ nsuf, int *__restrict__ nout) {
    __shared__ u32 mt[MT_N];
    const int c = blockIdx.x, lane = threadIdx.x;
    if (lane == 0) mt_seed(mt, syn_key(syn_key(syn_key(syn_key(RSIM_GOLDEN, seed), SYN_RNG_SALT), (u64)c), 1ull));
    __syncwarp();
    const SynClass C = cls[c];
    const u64 ns = (u64)(C.suf_hi - C.suf_lo) + 1, no = (u64)(C.out_hi - C.out_lo) + 1;
    const int ks = syn_bitlen(ns), ko = syn_bitlen(no);
    const i64 need = 2 * (coff[c + 1] - coff[c]);   // draws
    int *suf = nsuf + coff[c], *outp = nout + coff[c];
    i64 d = 0;                                      // draws accepted so far (state = d & 1)
    while (d < need) {
        mt_twist(mt, lane);
        for (int base = 0; base < MT_N && d < need; base += 32) {
            const int j = base + lane;
            const u32 w = j < MT_N ? mt_temper(mt[j]) : 0u;
            const u32 v0 = w >> (32 - ks), v1 = w >> (32 - ko);
            const bool a0 = j < MT_N && (u64)v0 < ns, a1 = j < MT_N && (u64)v1 < no;
            // map as 2 bits: bit s = image of state s
            u32 f = (a0 ? 1u : 0u) | ((a1 ? 0u : 1u) << 1);
            u32 pre = f;                            // inclusive scan: pre = f_lane o ... o f_0
            #pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const u32 g = __shfl_up_sync(FULL, pre, o);
                if (lane >= o) pre = ((pre >> ((g >> 0) & 1)) & 1) | (((pre >> ((g >> 1) & 1)) & 1) << 1);
            }
            u32 ex = __shfl_up_sync(FULL, pre, 1);  // exclusive: maps of the lanes before
            if (lane == 0) ex = 2u;                 // identity: 0 -> 0, 1 -> 1
            const int s0 = (int)(d & 1);
            const int st = (int)((ex >> s0) & 1);   // this lane's entry state
            const bool acc = st ? a1 : a0;
            const u32 ball = __ballot_sync(FULL, acc);
            const i64 di = d + __popc(ball & ((1u << lane) - 1u));
            if (acc && di < need) {
                if (st == 0) suf[di >> 1] = (int)(C.suf_lo + v0);
                else outp[di >> 1] = (int)(C.out_lo + v1);
            }
            d += __popc(ball);
        }
    }
}

// Thread per arrival (class c, seq s, time t): its index in the sorted (t, ci, seq) order is
// s + #{earlier classes' times <= t} + #{later classes' times < t}. Class c's times sit at
// times[toff[c] .. toff[c] + n_c), n_c = coff[c+1] - coff[c].
__global__ void synth_order_kernel(const SynClass *__restrict__ cls, int n_classes, const i64 *__restrict__ toff,
                                   const i64 *__restrict__ coff, const double *__restrict__ times, const int *__restrict__ nsuf,
                                   const int *__restrict__ nout, i64 total, double *__restrict__ arrival_s,
                                   int *__restrict__ row_cls, i64 *__restrict__ row_seq, i64 *__restrict__ row_len,
                                   i64 *__restrict__ row_out) {
    const i64 g = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= total) return;
    int c = 0;
    while (coff[c + 1] <= g) c++;
    const i64 s = g - coff[c];
    const double t = times[toff[c] + s];
    i64 rank = s;
    for (int o = 0; o < n_classes; o++) {
        if (o == c) continue;
        i64 lo = toff[o], hi = toff[o] + coff[o + 1] - coff[o];   // first time > t (o < c) / >= t
        while (lo < hi) {
            const i64 mid = (lo + hi) >> 1;
            const double v = times[mid];
            if (o < c ? v <= t : v < t) lo = mid + 1; else hi = mid;
        }
        rank += lo - toff[o];
    }
    arrival_s[rank] = t;
    row_cls[rank] = c;
    row_seq[rank] = s;
    row_len[rank] = cls[c].shared + nsuf[g];
    row_out[rank] = nout[g];
}

// Warp per request: blocks[blk_off[r] ..], class_key, input tokens, request id.
__global__ void synth_blocks_kernel(const SynClass *__restrict__ cls, u64 seed, i64 total, i64 block_size,
                                    const int *__restrict__ row_cls, const i64 *__restrict__ row_seq,
                                    const i64 *__restrict__ blk_off, u64 *__restrict__ blocks,
                                    u64 *__restrict__ request_id, i64 *__restrict__ in_tokens,
                                    u64 *__restrict__ class_key) {
    const i64 r = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= total) return;
    const int c = row_cls[r];
    const i64 sh = cls[c].shared, a = blk_off[r], len = blk_off[r + 1] - a;
    const u64 shared_acc = syn_key(syn_key(syn_key(RSIM_GOLDEN, seed), SYN_SHARED_SALT), (u64)c);
    const u64 suffix_acc = syn_key(syn_key(syn_key(syn_key(RSIM_GOLDEN, seed), SYN_SUFFIX_SALT), (u64)c),
                                   (u64)row_seq[r]);
    for (i64 p = lane; p < len; p += 32)
        __stcs(blocks + a + p, p < sh ? syn_key(shared_acc, (u64)p) : syn_key(suffix_acc, (u64)(p - sh)));
    if (lane == 0) {
        const u64 b0 = sh > 0 ? syn_key(shared_acc, 0) : syn_key(suffix_acc, 0);
        u64 ck = syn_key(syn_key(RSIM_GOLDEN, SYN_CLASS_SALT), b0);
        if (len >= 2) ck = syn_key(ck, sh > 1 ? syn_key(shared_acc, 1) : syn_key(suffix_acc, (u64)(1 - sh)));
        class_key[r] = ck;
        request_id[r] = (u64)r;
        in_tokens[r] = len * block_size;
    }
}
