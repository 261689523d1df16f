// rsim.cu -- librsim: host side of the C ABI declared in include/rsim.h.
//
// Owns all device memory of one GPU's instance shard, a CUDA stream and the
// launch configuration of the persistent replay cluster. Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -lineinfo
//        -Xcompiler -fPIC -shared -o librsim.so rsim.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cstdarg>
#include <vector>
#include <algorithm>
#include <mutex>

#include "../../include/rsim.h"
#include "rsim_kernels.cuh"
#ifndef RSIM_SLOT_MULT
#define RSIM_SLOT_MULT 8   // table slots >= 8/3 x expected keys at least: load <= 3/8
#endif
#ifndef RSIM_CENTRAL
#define RSIM_CENTRAL 1
#endif
#ifndef RSIM_TABLE_BUDGET
#define RSIM_TABLE_BUDGET (256ull << 20)   // all N tables at load <= 3/32 only within this (L2-friendly)
#endif
#ifndef RSIM_TABLE_MAX
#define RSIM_TABLE_MAX (8ull << 30)        // load <= 3/16 up to this much HBM, else down to <= 3/8
#endif
#include "rsim_check.cuh"
#include "rsim_api.cuh"
#include "rsim_synth.cuh"
#include <cub/device/device_scan.cuh>
#include <cmath>

namespace {

char g_create_err[512] = "";

template <typename T>
struct DevArr {
    T *p = nullptr;
    size_t cap = 0;
    void free_() { if (p) cudaFree(p); p = nullptr; cap = 0; }
    // grow keeping the first `keep` elements
    cudaError_t reserve(size_t n, size_t keep, cudaStream_t s) {
        if (n <= cap) return cudaSuccess;
        size_t nc = std::max(n, cap * 2 + 16);
        T *q = nullptr;
        cudaError_t e = cudaMalloc(&q, nc * sizeof(T));
        if (e != cudaSuccess) return e;
        if (p && keep) {
            e = cudaMemcpyAsync(q, p, keep * sizeof(T), cudaMemcpyDeviceToDevice, s);
            if (e != cudaSuccess) { cudaFree(q); return e; }
            cudaStreamSynchronize(s);
        }
        if (p) cudaFree(p);
        p = q; cap = nc;
        return cudaSuccess;
    }
};

}  // namespace

struct rsim {
    rsim_config cfg;
    char err[512];
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    int C = 1, W = 1, ipw = 1, per_cta = 1;
    size_t smem_bytes = 0;
    bool central = false;           // replay_kernel's central mode: one extra decider CTA
    bool route1 = false;            // rsim_route_request in one launch (route_kernel)
    bool no_rsm = getenv("RSIM_NO_SMEM_RUNNING") != nullptr;   // A/B switch: running lists stay in HBM
    int qlog2 = 0, slog2 = 0;
    i64 max_occ = 0;
    i64 R = 0, nblk = 0, nout = 0;       // loaded requests, blocks, output keys
    i64 launches = 0;
    float last_replay_ms = 0, last_k1_ms = 0, last_drain_ms = 0;
    // trace
    DevArr<i64> arrival, in_tok, out_tok, blk_off, ooff;
    DevArr<u64> rid, blocks, ckeys, okeys;
    DevArr<int> hit_blocks, chosen;
    DevArr<i64> hit_tokens, first_sched, first_token, finish, route_bs, dec_ns;
    // instances
    Inst *inst = nullptr;
    QEnt *qbuf = nullptr;
    REnt *rbuf = nullptr;
    u64 *tkeys = nullptr;
    Meta *tmeta = nullptr;
    u64 *tie = nullptr;
    int *errbuf = nullptr;
    int *flag = nullptr;
    i64 *log = nullptr;
    u64 *log_n = nullptr;
    i64 log_cap = 0;
    double *scores = nullptr;
    u64 *scratch_keys = nullptr;
    size_t scratch_cap = 0;
    i64 *scratch_res = nullptr;
    u64 *ctr = nullptr;            // device counters (Params.ctr)
    int N = 0, gbase = 0;          // local shard size, global id of local instance 0
    u64 *mbox = nullptr;           // multi-GPU mailbox [2 parity][8 ranks][RSIM_MBOX_W]
    u64 *peer[8] = {nullptr};
    bool peer_ipc[8] = {false};
    u64 epoch = 1;
    Run *runs = nullptr;
    int rlog2 = 0;
    HEnt *hring = nullptr;   // view-history rings (staleness > 0)
    int4 *simj = nullptr;    // simulate: per-warp lists of requests joining the TTFT replay's decode set
    int hlog2 = 0;
    // hotspot detector (rsim_detector.cuh): classes loaded by rsim_load_detector
    DevArr<int> dtid, dtw;
    DevArr<i64> dtex, dbk, drows;
    DevArr<u64> dtkey;
    DevArr<DTrack> dtr;
    i64 *dtot = nullptr, *dglob = nullptr;
    int dT = 0, dTs = 0, dbclog2 = 0;   // tracks, bucket-ring track stride, window bucket log2
    int det_next_track = -1, det_next_len = 0;   // rsim_detector_next: the next routed request's class
    u64 det_next_key = 0;
    i64 det_next_rows = 0;
    i64 drows_cap = 0;
    bool det_loaded = false;
    DevArr<i64> ddbg;
    DevArr<u64> arena;             // API-inserted chain keys (named by eviction runs)
    i64 narena = 0;
    unsigned short *crit = nullptr; // diagnostics: per (decision, warp) phase records
    std::vector<i64> order_breaks;  // loaded request indices whose arrival precedes the previous one
    i64 last_arrival = 0;
    std::vector<i64> api_segs;      // debug_checks: API-inserted chains (instance, arena offset, length)
    DevArr<i64> dsegs;
    DevArr<u32> seen;               // debug_checks: per-slot "named by a chain" bits
    DevArr<u32> dupmask;            // route() API: instances holding the request id (bitmap)
    const u32 *cur_dupmask = nullptr;
    i64 crit_cap = 0;
    // rsim_route_request: one mapped pinned block in each direction (the request in, the
    // decision + scores + device error word out), read / written by the kernels themselves
    i64 *rq_h = nullptr;            // pinned request block
    DevArr<i64> rq_dev;             // its device copy
    size_t rq_cap = 0;              // i64 words
    i64 *ro_h = nullptr, *ro_d = nullptr;
    i64 *log_pin = nullptr;         // rsim_read_step_log's pinned bounce buffer
};

static rsim_status fail(rsim_t *h, rsim_status st, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    if (h) vsnprintf(h->err, sizeof(h->err), fmt, ap);
    else vsnprintf(g_create_err, sizeof(g_create_err), fmt, ap);
    va_end(ap);
    return st;
}

#define CK(h, call)                                                                            \
    do {                                                                                       \
        cudaError_t _e = (call);                                                               \
        if (_e != cudaSuccess)                                                                 \
            return fail((h), RSIM_E_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(_e), \
                        __FILE__, __LINE__);                                                   \
    } while (0)

static int ilog2_ceil(i64 v) { int l = 0; while ((1LL << l) < v) l++; return l; }

static Params make_params(rsim_t *h) {
    Params P;
    memset(&P, 0, sizeof(P));
    P.arrival = h->arrival.p; P.in_tok = h->in_tok.p; P.out_tok = h->out_tok.p;
    P.blk_off = h->blk_off.p; P.ooff = h->ooff.p;
    P.rid = h->rid.p; P.ckeys = h->ckeys.p; P.okeys = h->okeys.p;
    P.hit_blocks = h->hit_blocks.p; P.chosen = h->chosen.p; P.hit_tokens = h->hit_tokens.p;
    P.first_sched = h->first_sched.p; P.first_token = h->first_token.p; P.finish = h->finish.p;
    P.route_bs = h->route_bs.p; P.dec_ns = h->dec_ns.p;
    P.N = h->N; P.C = h->C; P.W = h->W; P.ipw = h->ipw; P.per_cta = h->per_cta;
    P.central = h->central ? 1 : 0;
    P.bs = h->cfg.block_size; P.policy = h->cfg.policy; P.kv_ind = h->cfg.kv_indicator;
    P.kvw = h->cfg.kv_weight; P.bsn = h->cfg.bs_norm_cap; P.range_thr = h->cfg.range_threshold;
    P.bal_ind = h->cfg.balance_indicator; P.debug = h->cfg.debug_checks;
    P.cap = h->cfg.capacity_blocks; P.chunk = h->cfg.chunk_tokens; P.max_batch = h->cfg.max_batch_requests;
    P.pb = h->cfg.prefill_base_ms; P.pt = h->cfg.prefill_per_token_ms; P.db = h->cfg.decode_base_ms;
    P.ds = h->cfg.decode_per_seq_ms; P.dcc = h->cfg.decode_per_ctx_token_ms; P.qw = h->cfg.q_weight;
    P.inst = h->inst; P.qbuf = h->qbuf; P.qlog2 = h->qlog2; P.rbuf = h->rbuf;
    P.tkeys = h->tkeys; P.tmeta = h->tmeta; P.slog2 = h->slog2; P.max_occ = h->max_occ; P.empty = 0;
    P.tie = h->tie; P.err = h->errbuf;
    P.log = h->log; P.log_cap = h->log_cap; P.log_n = h->log_n;
    P.scores = nullptr;
    P.ctr = h->ctr;
    P.gbase = h->gbase; P.world = h->cfg.world > 1 ? h->cfg.world : 1; P.rank = h->cfg.rank;
    P.mbox = h->mbox;
    for (int i = 0; i < 8; i++) P.peer[i] = h->peer[i];
    P.epoch = h->epoch;
    P.runs = h->runs; P.rlog2 = h->rlog2; P.arena = h->arena.p;
    P.stal = h->cfg.staleness_us; P.hring = h->hring; P.hlog2 = h->hlog2;
    P.simj = h->simj;
    P.spb = h->cfg.sim_prefill_base_ms; P.spt = h->cfg.sim_prefill_per_token_ms; P.sdb = h->cfg.sim_decode_base_ms;
    P.sds = h->cfg.sim_decode_per_seq_ms; P.sdc = h->cfg.sim_decode_per_ctx_token_ms;
    P.dtid = (h->cfg.det_on && h->det_loaded) ? h->dtid.p : nullptr;
    P.dtw = h->dtw.p; P.dtex = h->dtex.p; P.dtkey = h->dtkey.p; P.dtr = h->dtr.p;
    P.dbk = h->dbk.p; P.dtot = h->dtot; P.dglob = h->dglob; P.drows = h->drows.p; P.drows_cap = h->drows_cap;
    P.dwin = h->cfg.det_window_s; P.dmult = h->cfg.det_consecutive_multiplier;
    P.dwin_i = (i64)h->cfg.det_window_s; P.dcool = (i64)(h->cfg.det_window_s * 1e6);
    P.dT = h->dT; P.dTs = h->dTs; P.dtopk = h->cfg.det_top_k_classes; P.dforce = h->cfg.det_mitigation == 1;
    P.dmean = h->cfg.det_compare_mean_non_holder; P.dbclog2 = h->dbclog2;
    P.ddbg = h->ddbg.p;
    P.dsm = (P.dtid != nullptr && h->dT <= RSIM_DET_SMEM_T &&
             h->smem_bytes + (size_t)h->dT * (sizeof(DTrack) + sizeof(u64)) <= 220 * 1024) ? 1 : 0;
    P.timeout_ns = (h->cfg.comm_timeout_ms > 0 ? h->cfg.comm_timeout_ms : 10000) * 1000000LL;
    P.crit = h->crit; P.crit_cap = h->crit_cap;
    return P;
}

static rsim_status decode_device_error(rsim_t *h, const int *e);
static rsim_status check_device_error(rsim_t *h) {
    int e[4];
    CK(h, cudaMemcpyAsync(e, h->errbuf, sizeof(e), cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    return decode_device_error(h, e);
}
// the device error word (errbuf: code, instance, detail); non-zero words are cleared for the next call
static rsim_status decode_device_error(rsim_t *h, const int *e) {
    if (e[0] == 0) return RSIM_OK;
    CK(h, cudaMemsetAsync(h->errbuf, 0, 4 * sizeof(int), h->stream));
    switch (e[0]) {
        case DEV_E_CACHE_FULL: return fail(h, RSIM_E_CACHE_FULL, "pinned blocks exceed capacity");
        case DEV_E_INVARIANT: {
            static const char *what[] = {"unpin of a chain that is not pinned / missing chain",
                "aggregates != recount (InstanceSim.reconcile)", "entry with depth < 1 or pin < 0",
                "occupancy counter != present entries", "occupancy over capacity",
                "entry depth != its chain position", "prefix closure violated (parent missing)",
                "parent older than child breaks LRU eviction safety", "pin must cover the path",
                "present key on no chain of the instance"};
            const int c = (e[2] >= 1 && e[2] <= 9) ? e[2] : 0;
            if (c) return fail(h, RSIM_E_INVARIANT, "instance %d: %s", e[1], what[c]);
            return fail(h, RSIM_E_INVARIANT, "%s", what[0]);
        }
        case DEV_E_QUEUE_OVERFLOW: return fail(h, RSIM_E_QUEUE_OVERFLOW, "instance queue ring full (queue_capacity=%d)", 1 << h->qlog2);
        case DEV_E_TABLE_FULL: return fail(h, RSIM_E_TABLE_FULL, "instance KV$ table over 3/4 load (slots=%d)", 1 << h->slog2);
        case DEV_E_RUNS_FULL: return fail(h, RSIM_E_TABLE_FULL, "instance LRU touch-run ring full (runs=%d)", 1 << h->rlog2);
        case 11: return fail(h, RSIM_E_NO_INSTANCES, "no instances to route to");
        case DEV_E_DUPLICATE: return fail(h, RSIM_E_DUPLICATE, "request already present on the chosen instance");
        case DEV_E_DETECTOR: return fail(h, RSIM_E_DETECTOR, "detector capacity exceeded (more than %d classes re-evaluated at once, or a window bucket ring overflow)", RSIM_DLMAX);
        case DEV_E_HISTORY_OVERFLOW: return fail(h, RSIM_E_HISTORY_OVERFLOW, "instance view-history ring full (history_capacity=%d)", 1 << h->hlog2);
        case DEV_E_COMM: return fail(h, RSIM_E_COMM, "timed out waiting for a peer rank's decision partial");
        default: return fail(h, RSIM_E_INVARIANT, "device error %d", e[0]);
    }
}

static Inst fresh_inst() {
    Inst s;
    memset(&s, 0, sizeof(s));
    s.next_step = RSIM_NONE; s.due = RSIM_NONE; s.next_finish = RSIM_NONE;
    s.hhead = 0; s.htail = 1;   // history = [(-inf, zero view)]
    return s;
}

static rsim_status det_reset(rsim_t *h, cudaStream_t s) {    // Detector.__init__ state
    if (!h->cfg.det_on || !h->det_loaded) return RSIM_OK;
    CK(h, cudaMemsetAsync(h->dtr.p, 0, (size_t)h->dT * sizeof(DTrack), s));
    const i64 g[DG_N] = {0, 0, 0, -1, 0, 0, 0, INT64_MIN, 0, 0, 0};
    static_assert(DG_N == 11, "detector scalars");
    CK(h, cudaMemcpyAsync(h->dglob, g, sizeof(g), cudaMemcpyHostToDevice, s));
    CK(h, cudaStreamSynchronize(s));
    return RSIM_OK;
}

static rsim_status init_state(rsim_t *h) {
    const int N = h->N;
    h->epoch += 1;
    std::vector<Inst> hs(N);
    for (auto &s : hs) s = fresh_inst();
    CK(h, cudaMemcpyAsync(h->inst, hs.data(), N * sizeof(Inst), cudaMemcpyHostToDevice, h->stream));
    h->det_loaded = false;                          // classes belong to a loaded trace
    const size_t slots = (size_t)N << h->slog2;
    CK(h, cudaMemsetAsync(h->tkeys, 0, slots * sizeof(u64), h->stream));   // EMPTY = 0
    CK(h, cudaMemsetAsync(h->tmeta, 0, slots * sizeof(Meta), h->stream));
    u64 tie[2] = {h->cfg.tie_seed_lo, h->cfg.tie_seed_hi};
    CK(h, cudaMemcpyAsync(h->tie, tie, sizeof(tie), cudaMemcpyHostToDevice, h->stream));
    CK(h, cudaMemsetAsync(h->errbuf, 0, 4 * sizeof(int), h->stream));
    CK(h, cudaMemsetAsync(h->log_n, 0, sizeof(u64), h->stream));
    CK(h, cudaMemsetAsync(h->ctr, 0, 48 * sizeof(u64), h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    h->R = 0; h->nblk = 0; h->nout = 0; h->narena = 0;
    h->api_segs.clear();
    h->order_breaks.clear();
    h->last_arrival = 0;
    // blk_off / ooff hold a leading 0
    CK(h, h->blk_off.reserve(1, 0, h->stream));
    CK(h, h->ooff.reserve(1, 0, h->stream));
    CK(h, cudaMemsetAsync(h->blk_off.p, 0, sizeof(i64), h->stream));
    CK(h, cudaMemsetAsync(h->ooff.p, 0, sizeof(i64), h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    return RSIM_OK;
}

extern "C" {

const char *rsim_last_error(const rsim_t *h) { return h ? h->err : g_create_err; }
size_t rsim_config_size(void) { return sizeof(rsim_config); }
int64_t rsim_launch_count(const rsim_t *h) { return h ? h->launches : 0; }

rsim_status rsim_create(const rsim_config *cfg, rsim_t **out) {
    if (!cfg || !out) return fail(nullptr, RSIM_E_INVALID, "null argument");
    *out = nullptr;
    if (cfg->struct_size != sizeof(rsim_config) || cfg->abi_version != RSIM_ABI_VERSION)
        return fail(nullptr, RSIM_E_INVALID, "rsim_config layout mismatch: struct_size %u / abi_version %u, "
                    "this librsim expects %zu / %d", cfg->struct_size, cfg->abi_version, sizeof(rsim_config),
                    RSIM_ABI_VERSION);
    const rsim_config &c = *cfg;
    if (c.n_instances < 1) return fail(nullptr, RSIM_E_INVALID, "n_instances must be >= 1");
    if (c.block_size < 1) return fail(nullptr, RSIM_E_INVALID, "block_size must be >= 1");
    if (c.capacity_blocks == 0 || c.capacity_blocks < -1) return fail(nullptr, RSIM_E_INVALID, "capacity_blocks must be >= 1 or -1");
    if (c.chunk_tokens < 1 || c.max_batch_requests < 1) return fail(nullptr, RSIM_E_INVALID, "chunk_tokens and max_batch_requests must be >= 1");
    if (c.policy < 0 || c.policy > 5) return fail(nullptr, RSIM_E_UNSUPPORTED, "policy %d not on the device path", c.policy);
    if (c.staleness_us < 0) return fail(nullptr, RSIM_E_INVALID, "staleness_us must be >= 0");
    if (c.det_on) {
        if (!(c.det_window_s > 0) || c.det_top_k_classes < 1 || c.det_class_key_blocks < 1 ||
            c.det_mitigation < 0 || c.det_mitigation > 1)
            return fail(nullptr, RSIM_E_INVALID, "invalid detector configuration");
        if (c.world > 1) return fail(nullptr, RSIM_E_UNSUPPORTED, "the hotspot detector is single-rank on the device path");
        if (c.det_window_s > 1e6) return fail(nullptr, RSIM_E_UNSUPPORTED, "detector window longer than 1e6 s");
    }
    if (c.prefill_base_ms < 0 || c.prefill_per_token_ms < 0 || c.decode_base_ms < 0 || c.decode_per_seq_ms < 0 ||
        c.decode_per_ctx_token_ms < 0)
        return fail(nullptr, RSIM_E_INVALID, "cost model coefficients must be non-negative");
    if (c.max_batch_requests > (1 << 20)) return fail(nullptr, RSIM_E_INVALID, "max_batch_requests too large");

    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return fail(nullptr, RSIM_E_CUDA, "no CUDA device available (librsim has no CPU fallback): %s",
                    cudaGetErrorString(e));
    if (c.device < 0 || c.device >= ndev) return fail(nullptr, RSIM_E_INVALID, "device %d out of range", c.device);
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, c.device);
    if (prop.major < 10) return fail(nullptr, RSIM_E_CUDA, "device %s (sm_%d%d) is not sm_100", prop.name, prop.major, prop.minor);

    rsim_t *h = new rsim_t();
    h->cfg = c;
    h->err[0] = 0;
    if (cudaSetDevice(c.device) != cudaSuccess) { delete h; return fail(nullptr, RSIM_E_CUDA, "cudaSetDevice failed"); }
    CK(nullptr, cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    CK(nullptr, cudaEventCreate(&h->ev0));
    CK(nullptr, cudaEventCreate(&h->ev1));

    // ---- replay cluster shape
    const int world = c.world > 1 ? c.world : 1;
    if (world > 8 || c.rank < 0 || c.rank >= world) { delete h; return fail(nullptr, RSIM_E_INVALID, "world must be 1..8 and 0 <= rank < world"); }
    if (c.n_instances < world) { delete h; return fail(nullptr, RSIM_E_INVALID, "fewer instances than ranks"); }
    {   // contiguous shard of this rank (paper_2603_15202_b200/sharding.py: shard_bounds)
        const int base = c.n_instances / world, extra = c.n_instances % world;
        h->gbase = c.rank * base + std::min(c.rank, extra);
        h->N = base + (c.rank < extra ? 1 : 0);
    }
    const int N = h->N;
    // the extended kernel (launch_replay's choice); the plain one runs with a central decider CTA
    // (replay_kernel: central mode) when the instance shard still fits 15 CTAs
    const bool ext = c.policy == RSIM_POLICY_FILTER || (c.policy == RSIM_POLICY_LINEAR && !(c.bs_norm_cap > 0)) ||
                     c.staleness_us > 0 || c.det_on || c.policy == RSIM_POLICY_SIMULATE;
    int C = 0, per_cta = 0, W = 0, ipw = 0;
    auto shape = [&](int cmax) {
        C = c.ctas;
        if (C <= 0) C = std::min(cmax, N);     // measured: spreading instances over SMs wins (profiles/)
        C = std::max(1, std::min(cmax, std::min(C, N)));
        per_cta = (N + C - 1) / C;
        // default: the lean kernel (<= 7 instance warps, 255 registers) unless a warp would own > 32 instances
        W = c.warps_per_cta > 0 ? c.warps_per_cta : std::min(RSIM_LEAN_WARPS, per_cta);
        if (c.warps_per_cta <= 0 && (per_cta + W - 1) / W > 32) W = std::min(RSIM_MAX_WARPS, per_cta);
        W = std::max(1, std::min(RSIM_MAX_WARPS, W));
        ipw = (per_cta + W - 1) / W;
    };
    // (one CTA: up to 256 instances; a larger shard probes faster spread over the replay cluster)
    h->route1 = !ext && world == 1 && N <= 256 && !getenv("RSIM_ROUTE_3LAUNCH");
    h->central = false;
    if (!ext && RSIM_CENTRAL && !getenv("RSIM_NO_CENTRAL") && c.ctas <= 15) {
        shape(15);
        h->central = ipw <= 32;
    }
    if (!h->central) shape(16);
    if (ipw > 32) { delete h; return fail(nullptr, RSIM_E_INVALID, "too many instances per GPU (%d per warp > 32)", ipw); }
    if (C * W > 128) { delete h; return fail(nullptr, RSIM_E_INVALID, "cluster too large"); }   // decide_phase: <= 4 rounds of 32
    h->C = C; h->W = W; h->ipw = ipw; h->per_cta = per_cta;
    h->smem_bytes = (size_t)per_cta * sizeof(Inst) + (size_t)(6 * W * C) * sizeof(Part) + RSIM_SLOTS * sizeof(ReqStage) + 2 * sizeof(Dec) + 8 * sizeof(u64) + RSIM_MODTAB * sizeof(u32) + (size_t)W * sizeof(WarpBuf) +
                     (c.staleness_us > 0 ? (size_t)per_cta * sizeof(HistHead) : 0) +
                     (c.det_on ? sizeof(DetCtl) + (size_t)(8 * W * C) * sizeof(Part) + (size_t)(2 * W * C) * RSIM_DLMAX : 0);
    if (h->smem_bytes > 220 * 1024) { delete h; return fail(nullptr, RSIM_E_INVALID, "instance shard does not fit in shared memory"); }
    {   // kernel attributes are process-global: set the ceiling once (handles on other threads launch concurrently)
        static std::once_flag once;
        std::call_once(once, [] {
            const void *ks[] = {(const void *)replay_kernel<RSIM_LEAN_WARPS, false>, (const void *)replay_kernel<RSIM_MAX_WARPS, false>,
                                (const void *)replay_kernel<RSIM_LEAN_WARPS, true>, (const void *)replay_kernel<RSIM_MAX_WARPS, true>};
            for (const void *k : ks) {
                cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
                cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            }
            cudaFuncSetAttribute((const void *)route_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        });
    }

    // ---- sizing
    int ql = c.queue_capacity > 0 ? ilog2_ceil(c.queue_capacity) : 10;
    h->qlog2 = std::max(4, ql);
    int sl = c.table_slots_log2;
    if (sl <= 0) {
        i64 expect = c.expected_keys > 0 ? c.expected_keys : 3000;   // callers size from the trace
        // A low load factor keeps nearly every lookup inside the aligned 16-B slot pair at its
        // home (linear probing: a miss at load a scans ~(1 + 1/(1-a)^2)/2 slots). Load <= 3/32
        // while the N tables (24 B per slot) stay within RSIM_TABLE_BUDGET, else <= 3/8
        // (A/B on one B200, us/decision at load <= 3/4, 3/8, 3/16, 3/32: api64 6.05 / 5.20 /
        // 4.95 / 4.88; chat1024 7.07 / 6.80 / 6.71 / 6.82 -- but 3.2x the algorithmic DRAM bytes
        // at 3/32 (805 MB of tables); agent256 - / 19.1 / 18.4 / 18.3; large4096 12.7 / 12.2 /
        // 12.9 / 13.4).
        // Shards of more than 2048 instances keep 3/16 while the tables fit RSIM_TABLE_MAX and
        // 1 MB per instance (large4096, 1M requests: 15.97 us/decision at load <= 3/8 in 400 MB
        // of tables, 15.12 at <= 3/16 in 3.2 GB). Smaller shards go to 3/8: chat1024 at 3/16
        // replays no faster and moves 10.1 GB of DRAM per launch instead of 1.6 GB
        // (profiles/r2_ab/traffic_chat1024_tables_2p14.csv); agent256's 3 MB tables at 3/16
        // replay 3 % faster but halve the what-if probe's throughput.
        int mult = 32;
        sl = ilog2_ceil(expect * mult / 3 + 64);
        auto tab_bytes = [&] { return ((size_t)N << sl) * 24; };
        const bool over = tab_bytes() > (size_t)RSIM_TABLE_BUDGET;   // (tables within it keep 3/32)
        const int floor16 = N > 2048 ? 16 : RSIM_SLOT_MULT;
        while (mult > floor16 && tab_bytes() > (size_t)RSIM_TABLE_BUDGET) {
            mult /= 2;
            sl = ilog2_ceil(expect * mult / 3 + 64);
        }
        while (over && mult > RSIM_SLOT_MULT && (tab_bytes() > (size_t)RSIM_TABLE_MAX || (24ull << sl) > (1ull << 20))) {
            mult /= 2;
            sl = ilog2_ceil(expect * mult / 3 + 64);
        }
    }
    h->slog2 = std::max(6, std::min(30, sl));
    h->max_occ = ((i64)3 << h->slog2) / 4;
    const size_t slots = (size_t)N << h->slog2;
    CK(nullptr, cudaMalloc(&h->inst, N * sizeof(Inst)));
    CK(nullptr, cudaMalloc(&h->qbuf, ((size_t)N << h->qlog2) * sizeof(QEnt)));
    CK(nullptr, cudaMalloc(&h->rbuf, (size_t)N * c.max_batch_requests * sizeof(REnt)));
    CK(nullptr, cudaMalloc(&h->tkeys, slots * sizeof(u64)));
    CK(nullptr, cudaMalloc(&h->tmeta, slots * sizeof(Meta)));
    if (c.capacity_blocks > 0) {   // touch-run rings for exact LRU eviction (rsim_lru.cuh)
        const i64 want = c.runs_capacity > 0 ? c.runs_capacity : 4 * (1LL << h->qlog2) + 1024;
        h->rlog2 = std::max(6, std::min(26, ilog2_ceil(want)));
        CK(nullptr, cudaMalloc(&h->runs, ((size_t)N << h->rlog2) * sizeof(Run)));
    }
    if (c.staleness_us > 0) {   // view-history rings (indicators.py:36-65)
        h->hlog2 = std::max(4, std::min(24, ilog2_ceil(c.history_capacity > 0 ? c.history_capacity : 1024)));
        CK(nullptr, cudaMalloc(&h->hring, ((size_t)N << h->hlog2) * sizeof(HEnt)));
    }
    if (c.policy == RSIM_POLICY_SIMULATE)   // <= one joined entry per queued request ahead of the candidate
        CK(nullptr, cudaMalloc(&h->simj, ((size_t)(h->C * h->W) << h->qlog2) * sizeof(int4)));
    CK(nullptr, cudaMalloc(&h->tie, 2 * sizeof(u64)));
    CK(nullptr, cudaMalloc(&h->errbuf, 4 * sizeof(int)));
    CK(nullptr, cudaMalloc(&h->flag, sizeof(int)));
    CK(nullptr, cudaMalloc(&h->log_n, sizeof(u64)));
    // [N..2N): filter's second branch; with the detector, for route(): [2N..3N) batch sizes (least_bs),
    // [3N..4N) holders of the request's class, [4N..5N) kept-set scores, [5N] the verdict's branch
    CK(nullptr, cudaMalloc(&h->scores, (5 * (size_t)N + 1) * sizeof(double)));
    CK(nullptr, cudaMalloc(&h->scratch_res, 4 * sizeof(i64)));
    CK(nullptr, cudaMalloc(&h->ctr, 48 * sizeof(u64)));   // [16..47]: diagnostics builds
    CK(nullptr, cudaMalloc(&h->mbox, 2 * 8 * RSIM_MBOX_W * sizeof(u64)));
    CK(nullptr, cudaMemset(h->mbox, 0, 2 * 8 * RSIM_MBOX_W * sizeof(u64)));
    h->peer[world > 1 ? c.rank : 0] = h->mbox;
    if (c.record_steps) {
        h->log_cap = c.step_log_capacity > 0 ? c.step_log_capacity : (1 << 20);
        CK(nullptr, cudaMalloc(&h->log, (size_t)h->log_cap * 6 * sizeof(i64)));
    }
    rsim_status st = init_state(h);
    if (st != RSIM_OK) { snprintf(g_create_err, sizeof(g_create_err), "%s", h->err); rsim_destroy(h); return st; }
    *out = h;
    return RSIM_OK;
}

void rsim_destroy(rsim_t *h) {
    if (!h) return;
    cudaSetDevice(h->cfg.device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    DevArr<i64> *ai[] = {&h->arrival, &h->in_tok, &h->out_tok, &h->blk_off, &h->ooff, &h->hit_tokens,
                         &h->first_sched, &h->first_token, &h->finish, &h->route_bs, &h->dec_ns};
    for (auto *a : ai) a->free_();
    h->rid.free_(); h->blocks.free_(); h->ckeys.free_(); h->okeys.free_();
    h->hit_blocks.free_(); h->chosen.free_();
    void *ps[] = {h->inst, h->qbuf, h->rbuf, h->tkeys, h->tmeta, h->tie, h->errbuf, h->flag, h->log, h->log_n,
                  h->scores, h->scratch_keys, h->scratch_res, h->ctr, h->mbox, h->runs, h->crit, h->hring,
                  h->dtot, h->dglob, h->simj};
    h->dsegs.free_(); h->seen.free_(); h->dupmask.free_();
    if (h->rq_h) cudaFreeHost(h->rq_h);
    if (h->ro_h) cudaFreeHost(h->ro_h);
    if (h->log_pin) cudaFreeHost(h->log_pin);
    h->log_pin = nullptr;
    h->rq_h = h->ro_h = h->ro_d = nullptr; h->rq_cap = 0;
    h->rq_dev.free_();
    h->ddbg.free_(); h->dtid.free_(); h->dtw.free_(); h->dtex.free_(); h->dbk.free_(); h->drows.free_(); h->dtkey.free_(); h->dtr.free_();
    h->arena.free_();
    for (int i = 0; i < 8; i++) if (h->peer_ipc[i] && h->peer[i]) cudaIpcCloseMemHandle(h->peer[i]);
    for (void *p : ps) if (p) cudaFree(p);
    if (h->ev0) cudaEventDestroy(h->ev0);
    if (h->ev1) cudaEventDestroy(h->ev1);
    if (h->stream) cudaStreamDestroy(h->stream);
    delete h;
}

rsim_status rsim_reset(rsim_t *h) {
    if (!h) return RSIM_E_INVALID;
    CK(h, cudaSetDevice(h->cfg.device));
    return init_state(h);
}

rsim_status rsim_load_trace(rsim_t *h, int64_t n, const int64_t *arrival_us, const int64_t *input_tokens,
                            const int64_t *output_tokens, const uint64_t *request_id, const int64_t *blk_off,
                            const uint64_t *blocks) {
    if (!h) return RSIM_E_INVALID;
    if (n < 0) return fail(h, RSIM_E_INVALID, "negative request count");
    if (n == 0) return RSIM_OK;
    if (!arrival_us || !input_tokens || !output_tokens || !request_id || !blk_off || !blocks)
        return fail(h, RSIM_E_INVALID, "null trace array");
    CK(h, cudaSetDevice(h->cfg.device));
    if (blk_off[0] != 0) return fail(h, RSIM_E_TRACE, "blk_off[0] must be 0");
    const i64 bs = h->cfg.block_size;
    std::vector<i64> off(n + 1), oo(n + 1);
    oo[0] = h->nout;
    for (i64 i = 0; i < n; i++) {
        const i64 B = blk_off[i + 1] - blk_off[i];
        if (B < 1) return fail(h, RSIM_E_TRACE, "request %lld has no blocks", (long long)i);
        if (input_tokens[i] < 1 || output_tokens[i] < 1) return fail(h, RSIM_E_TRACE, "request %lld: in/out must be >= 1", (long long)i);
        if (input_tokens[i] > (1LL << 40) || output_tokens[i] > (1LL << 31)) return fail(h, RSIM_E_TRACE, "request %lld: token count too large", (long long)i);
        if (i > 0 && arrival_us[i] < arrival_us[i - 1]) return fail(h, RSIM_E_TRACE, "arrivals are not sorted");
        off[i] = h->nblk + blk_off[i];
        oo[i + 1] = oo[i] + (output_tokens[i] + bs - 1) / bs;
    }
    off[n] = h->nblk + blk_off[n];
    // route()/enqueue() API requests may arrive at any time; a replay range must not span an
    // arrival that precedes its predecessor (rsim_replay checks against these breaks)
    if (h->R > 0 && arrival_us[0] < h->last_arrival) h->order_breaks.push_back(h->R);
    h->last_arrival = arrival_us[n - 1];
    const i64 R0 = h->R, R1 = h->R + n, nb = blk_off[n], no = oo[n] - h->nout;
    cudaStream_t s = h->stream;
    CK(h, h->arrival.reserve(R1, R0, s)); CK(h, h->in_tok.reserve(R1, R0, s)); CK(h, h->out_tok.reserve(R1, R0, s));
    CK(h, h->rid.reserve(R1, R0, s)); CK(h, h->blk_off.reserve(R1 + 1, R0 + 1, s)); CK(h, h->ooff.reserve(R1 + 1, R0 + 1, s));
    CK(h, h->blocks.reserve(h->nblk + nb, h->nblk, s)); CK(h, h->ckeys.reserve(h->nblk + nb, h->nblk, s));
    CK(h, h->okeys.reserve(h->nout + no + 1, h->nout, s));
    CK(h, h->hit_blocks.reserve(R1, R0, s)); CK(h, h->chosen.reserve(R1, R0, s));
    DevArr<i64> *outs[] = {&h->hit_tokens, &h->first_sched, &h->first_token, &h->finish, &h->route_bs, &h->dec_ns};
    for (auto *a : outs) CK(h, a->reserve(R1, R0, s));
    CK(h, cudaMemcpyAsync(h->arrival.p + R0, arrival_us, n * sizeof(i64), cudaMemcpyHostToDevice, s));
    CK(h, cudaMemcpyAsync(h->in_tok.p + R0, input_tokens, n * sizeof(i64), cudaMemcpyHostToDevice, s));
    CK(h, cudaMemcpyAsync(h->out_tok.p + R0, output_tokens, n * sizeof(i64), cudaMemcpyHostToDevice, s));
    CK(h, cudaMemcpyAsync(h->rid.p + R0, request_id, n * sizeof(u64), cudaMemcpyHostToDevice, s));
    CK(h, cudaMemcpyAsync(h->blk_off.p + R0, off.data(), (n + 1) * sizeof(i64), cudaMemcpyHostToDevice, s));
    CK(h, cudaMemcpyAsync(h->ooff.p + R0, oo.data(), (n + 1) * sizeof(i64), cudaMemcpyHostToDevice, s));
    CK(h, cudaMemcpyAsync(h->blocks.p + h->nblk, blocks, nb * sizeof(u64), cudaMemcpyHostToDevice, s));
    for (auto *a : outs) CK(h, cudaMemsetAsync(a->p + R0, 0xff, n * sizeof(i64), s));   // -1
    CK(h, cudaMemsetAsync(h->chosen.p + R0, 0xff, n * sizeof(int), s));
    CK(h, cudaMemsetAsync(h->hit_blocks.p + R0, 0, n * sizeof(int), s));
    CK(h, cudaMemsetAsync(h->flag, 0, sizeof(int), s));
    // K1
    const i64 nwarps = (n + 31) / 32;
    const int grid = (int)((nwarps + K1_WARPS - 1) / K1_WARPS);
    CK(h, cudaEventRecord(h->ev0, s));
    k1_chain_keys<<<grid, 32 * K1_WARPS, 0, s>>>(h->blk_off.p, h->blocks.p, h->ckeys.p, h->ooff.p, h->okeys.p,
                                                   h->rid.p, R0, R1, 0ULL, h->flag);
    h->launches++;
    CK(h, cudaGetLastError());
    CK(h, cudaEventRecord(h->ev1, s));
    int flag = 0;
    CK(h, cudaMemcpyAsync(&flag, h->flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(h, cudaStreamSynchronize(s));
    cudaEventElapsedTime(&h->last_k1_ms, h->ev0, h->ev1);
    h->R = R1; h->nblk += nb; h->nout += no;
    if (flag) return fail(h, RSIM_E_TRACE, "a chain key equals the table sentinel 0 (probability 2^-64 per key)");
    return RSIM_OK;
}

static rsim_status launch_replay(rsim_t *h, i64 k0, i64 k1, i64 until, int mode, int target, double *scores_dev,
                                 float *ms_out, bool sync = true) {
    if (h->cfg.world > 1) {
        if (mode == MODE_ROUTE || mode == MODE_ENQUEUE)
            return fail(h, RSIM_E_UNSUPPORTED, "route/enqueue API calls are single-rank only");
        for (int r = 0; r < h->cfg.world; r++)
            if (!h->peer[r]) return fail(h, RSIM_E_COMM, "peer mailbox of rank %d not set", r);
    }
    Params P = make_params(h);
    P.scores = scores_dev;
    P.dupmask = h->cur_dupmask;
    if (P.dtid != nullptr && !P.dsm && h->C > 1)
        return fail(h, RSIM_E_DETECTOR, "%d detector classes do not fit in shared memory next to the instance shard; "
                    "use ctas=1", h->dT);
    cudaLaunchConfig_t lc;
    memset(&lc, 0, sizeof(lc));
    const int cs = h->C + (h->central ? 1 : 0);    // + the decider CTA
    lc.gridDim = dim3(cs, 1, 1);
    lc.blockDim = dim3(32 * (h->W + 1), 1, 1);   // + the control warp
    lc.dynamicSmemBytes = h->smem_bytes + (P.dsm ? (size_t)h->dT * (sizeof(DTrack) + sizeof(u64)) : 0);
    {   // small shards keep their running lists in shared memory for the launch
        const size_t rs = (size_t)h->per_cta * (size_t)h->cfg.max_batch_requests * sizeof(REnt);
        const size_t off = (lc.dynamicSmemBytes + 127) & ~(size_t)127;
        if (!h->no_rsm && off + rs <= 220 * 1024) { P.rsm_off = (int)off; lc.dynamicSmemBytes = off + rs; }
    }
    lc.stream = h->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    if (sync) CK(h, cudaEventRecord(h->ev0, h->stream));
    const bool filt = h->cfg.policy == RSIM_POLICY_FILTER ||            // the extended kernel: two-branch or
                      (h->cfg.policy == RSIM_POLICY_LINEAR && !(h->cfg.bs_norm_cap > 0)) ||   // two-round decisions,
                      h->cfg.staleness_us > 0 || h->cfg.det_on ||                           // stale snapshots, detector,
                      h->cfg.policy == RSIM_POLICY_SIMULATE;                                // TTFT replays
    if (h->W <= RSIM_LEAN_WARPS && !filt)
        CK(h, cudaLaunchKernelEx(&lc, replay_kernel<RSIM_LEAN_WARPS, false>, P, (i64)k0, (i64)k1, (i64)until, mode, target));
    else if (!filt)
        CK(h, cudaLaunchKernelEx(&lc, replay_kernel<RSIM_MAX_WARPS, false>, P, (i64)k0, (i64)k1, (i64)until, mode, target));
    else if (h->W <= RSIM_LEAN_WARPS)
        CK(h, cudaLaunchKernelEx(&lc, replay_kernel<RSIM_LEAN_WARPS, true>, P, (i64)k0, (i64)k1, (i64)until, mode, target));
    else
        CK(h, cudaLaunchKernelEx(&lc, replay_kernel<RSIM_MAX_WARPS, true>, P, (i64)k0, (i64)k1, (i64)until, mode, target));
    h->launches++;
    if (!sync) return RSIM_OK;       // rsim_route_request: the caller collects results + error word
    CK(h, cudaEventRecord(h->ev1, h->stream));
    CK(h, cudaEventSynchronize(h->ev1));
    if (ms_out) cudaEventElapsedTime(ms_out, h->ev0, h->ev1);
    return check_device_error(h);
}

// debug_checks (cluster.py:168-170): reconcile + check_invariants of every instance on device
static rsim_status run_checks(rsim_t *h) {
    const size_t words = (((size_t)h->N << h->slog2) + 31) / 32;
    CK(h, h->seen.reserve(words, 0, h->stream));
    CK(h, cudaMemsetAsync(h->seen.p, 0, words * sizeof(u32), h->stream));
    const i64 nseg = (i64)h->api_segs.size() / 3;
    CK(h, h->dsegs.reserve(h->api_segs.size() + 3, 0, h->stream));
    if (nseg) CK(h, cudaMemcpyAsync(h->dsegs.p, h->api_segs.data(), h->api_segs.size() * sizeof(i64),
                                    cudaMemcpyHostToDevice, h->stream));
    const int threads = 128, blocks = (h->N * 32 + threads - 1) / threads;
    check_invariants_kernel<<<blocks, threads, 0, h->stream>>>(make_params(h), h->R, h->dsegs.p, nseg, h->seen.p);
    h->launches++;
    CK(h, cudaGetLastError());
    return check_device_error(h);
}

rsim_status rsim_replay(rsim_t *h, int64_t first, int64_t count) {
    if (!h) return RSIM_E_INVALID;
    if (first < 0 || count < 0 || first + count > h->R) return fail(h, RSIM_E_INVALID, "decision range out of the loaded trace");
    if (count == 0) return RSIM_OK;
    for (i64 b : h->order_breaks)
        if (b > first && b < first + count) return fail(h, RSIM_E_TRACE, "replay range spans unsorted arrivals");
    CK(h, cudaSetDevice(h->cfg.device));
    if (h->cfg.debug_checks) {      // one decision per launch, the checks after each (its steps ran before it)
        float tot = 0;
        for (i64 k = first; k < first + count; k++) {
            rsim_status st = launch_replay(h, k, k + 1, 0, MODE_REPLAY, -1, nullptr, &h->last_replay_ms);
            if (st) return st;
            tot += h->last_replay_ms;
            if ((st = run_checks(h))) return st;
        }
        h->last_replay_ms = tot;
        return RSIM_OK;
    }
    return launch_replay(h, first, first + count, 0, MODE_REPLAY, -1, nullptr, &h->last_replay_ms);
}

rsim_status rsim_drain(rsim_t *h, int64_t until_us) {
    if (!h) return RSIM_E_INVALID;
    CK(h, cudaSetDevice(h->cfg.device));
    rsim_status st = launch_replay(h, 0, 0, until_us, MODE_DRAIN, -1, nullptr, &h->last_drain_ms);
    if (st == RSIM_OK && h->cfg.debug_checks) st = run_checks(h);
    return st;
}
rsim_status rsim_check_invariants(rsim_t *h) {
    if (!h) return RSIM_E_INVALID;
    CK(h, cudaSetDevice(h->cfg.device));
    return run_checks(h);
}
rsim_status rsim_debug_corrupt(rsim_t *h, int32_t instance, int32_t what) {
    if (!h) return RSIM_E_INVALID;
    if (instance < 0 || instance >= h->N || what < 0 || what > 2) return fail(h, RSIM_E_INVALID, "bad fault");
    CK(h, cudaSetDevice(h->cfg.device));
    debug_corrupt_kernel<<<1, 32, 0, h->stream>>>(make_params(h), instance, what);
    h->launches++;
    CK(h, cudaGetLastError());
    CK(h, cudaStreamSynchronize(h->stream));
    return RSIM_OK;
}

rsim_status rsim_route_one(rsim_t *h, int64_t r, int64_t now_us, int32_t *chosen, int64_t *hit_tokens, double *scores) {
    return rsim_route_one_excl(h, r, now_us, nullptr, 0, chosen, hit_tokens, scores);
}
rsim_status rsim_route_one_excl(rsim_t *h, int64_t r, int64_t now_us, const int32_t *holders, int32_t n_holders,
                                int32_t *chosen, int64_t *hit_tokens, double *scores) {
    if (!h) return RSIM_E_INVALID;
    if (h->cfg.det_on) return fail(h, RSIM_E_UNSUPPORTED, "route/enqueue API calls with the hotspot detector: use a trace replay");
    if (r < 0 || r >= h->R) return fail(h, RSIM_E_INVALID, "request index out of range");
    CK(h, cudaSetDevice(h->cfg.device));
    const u32 *dm = nullptr;
    if (n_holders > 0) {
        const size_t words = ((size_t)h->cfg.n_instances + 31) / 32;
        std::vector<u32> m(words, 0u);
        for (int i = 0; i < n_holders; i++) {
            if (holders[i] < 0 || holders[i] >= h->cfg.n_instances) return fail(h, RSIM_E_INVALID, "holder out of range");
            m[holders[i] >> 5] |= 1u << (holders[i] & 31);
        }
        CK(h, h->dupmask.reserve(words, 0, h->stream));
        CK(h, cudaMemcpy(h->dupmask.p, m.data(), words * sizeof(u32), cudaMemcpyHostToDevice));
        dm = h->dupmask.p;
    }
    h->cur_dupmask = dm;
    rsim_status st = launch_replay(h, r, r + 1, now_us, MODE_ROUTE, -1, scores ? h->scores : nullptr, nullptr);
    h->cur_dupmask = nullptr;
    if (st != RSIM_OK) return st;
    if (chosen) CK(h, cudaMemcpy(chosen, h->chosen.p + r, sizeof(int), cudaMemcpyDeviceToHost));
    if (hit_tokens) CK(h, cudaMemcpy(hit_tokens, h->hit_tokens.p + r, sizeof(i64), cudaMemcpyDeviceToHost));
    if (scores) {
        CK(h, cudaMemcpy(scores, h->scores, h->N * sizeof(double), cudaMemcpyDeviceToHost));
        if (h->cfg.policy == RSIM_POLICY_FILTER) {   // the branch route_filter took (policies.py:180-183)
            std::vector<double> bsv(h->N);
            CK(h, cudaMemcpy(bsv.data(), h->scores + h->N, h->N * sizeof(double), cudaMemcpyDeviceToHost));
            const auto mm = std::minmax_element(bsv.begin(), bsv.end());
            if ((i64)*mm.second - (i64)*mm.first > h->cfg.range_threshold)
                memcpy(scores, bsv.data(), h->N * sizeof(double));
        }
    }
    return RSIM_OK;
}

// Detector state for route() API calls, grown in place: per-request track ids for R requests,
// T tracks (new ones zeroed; the per-CTA bucket rings re-laid out when the track stride grows,
// doubling) and room for `rows` DetectorRows. The first call initialises (Detector.__init__).
static rsim_status det_ensure(rsim_t *h, int T, i64 R, i64 rows) {
    cudaStream_t s = h->stream;
    int bl = 0;
    while ((1LL << bl) < (i64)h->cfg.det_window_s + 2) bl++;
    const bool first = !h->det_loaded;
    const int T0 = first ? 0 : h->dT;
    if (!first && bl != h->dbclog2) return fail(h, RSIM_E_DETECTOR, "detector window changed");
    CK(h, h->dtid.reserve(R, first ? 0 : h->R, s));
    if (T > T0) {
        CK(h, h->dtw.reserve(T, T0, s)); CK(h, h->dtex.reserve(T, T0, s)); CK(h, h->dtkey.reserve(T, T0, s));
        CK(h, h->dtr.reserve(T, T0, s));
        CK(h, cudaMemsetAsync(h->dtr.p + T0, 0, (size_t)(T - T0) * sizeof(DTrack), s));
        if (T > h->dTs) {                                   // bucket rings [C][stride][3 << bl]
            const int ns = std::max(T, 2 * h->dTs + 8);
            const size_t ring = (size_t)3 << bl;
            i64 *nb = nullptr;
            CK(h, cudaMalloc(&nb, (size_t)ns * ring * h->C * sizeof(i64)));
            if (h->dTs > 0 && h->dbk.p)
                CK(h, cudaMemcpy2DAsync(nb, (size_t)ns * ring * sizeof(i64), h->dbk.p, (size_t)h->dTs * ring * sizeof(i64),
                                        (size_t)h->dTs * ring * sizeof(i64), h->C, cudaMemcpyDeviceToDevice, s));
            CK(h, cudaStreamSynchronize(s));
            h->dbk.free_();
            h->dbk.p = nb; h->dbk.cap = (size_t)ns * ring * h->C;
            h->dTs = ns;
        }
    }
    if (rows > h->drows_cap) {
        CK(h, h->drows.reserve((size_t)rows * 7, (size_t)h->drows_cap * 7, s));
        h->drows_cap = rows;
    }
    if (!h->dtot || bl > h->dbclog2) {
        if (h->dtot) cudaFree(h->dtot);
        CK(h, cudaMalloc(&h->dtot, ((size_t)2 << bl) * h->C * sizeof(i64)));
    }
    if (!h->dglob) CK(h, cudaMalloc(&h->dglob, DG_N * sizeof(i64)));
    h->dT = std::max(T, T0); h->dbclog2 = bl;
    if (first) {
        h->det_loaded = true;
        return det_reset(h, s);
    }
    return RSIM_OK;
}

rsim_status rsim_detector_next(rsim_t *h, int32_t track, int32_t exemplar_len, uint64_t class_key,
                               int64_t rows_capacity) {
    if (!h) return RSIM_E_INVALID;
    if (!h->cfg.det_on) return fail(h, RSIM_E_INVALID, "handle was created without a detector");
    const int T0 = h->det_loaded ? h->dT : 0;
    if (track < 0 || track > T0) return fail(h, RSIM_E_INVALID, "track ids must be numbered by first arrival");
    if (track == T0 && exemplar_len < 1) return fail(h, RSIM_E_INVALID, "bad exemplar length");
    h->det_next_track = track; h->det_next_len = exemplar_len; h->det_next_key = class_key;
    h->det_next_rows = std::max<i64>(rows_capacity, 16);
    return RSIM_OK;
}

// ClusterSim.route(record, now_us) of a request that is not loaded yet (cluster.py:130-154): the
// request is appended to the device trace by route_ingest_kernel straight from mapped pinned
// memory, decided by a one-decision replay launch, and the decision + scores + device error word
// come back through mapped memory written by route_out_kernel: three launches, one synchronisation.
rsim_status rsim_route_request(rsim_t *h, int64_t now_us, int64_t input_tokens, int64_t output_tokens,
                               uint64_t request_id, const uint64_t *blocks, int64_t n_blocks,
                               const int32_t *holders, int32_t n_holders, int32_t *chosen, int64_t *hit_tokens,
                               double *scores, int32_t *branch) {
    if (!h) return RSIM_E_INVALID;
    if (h->cfg.det_on && h->det_next_track < 0)
        return fail(h, RSIM_E_INVALID, "route() with the hotspot detector: rsim_detector_next names the request's class first");
    if (h->cfg.world > 1) return fail(h, RSIM_E_UNSUPPORTED, "route/enqueue API calls are single-rank only");
    if (n_blocks < 1 || !blocks) return fail(h, RSIM_E_TRACE, "request has no blocks");
    if (input_tokens < 1 || output_tokens < 1) return fail(h, RSIM_E_TRACE, "request: in/out must be >= 1");
    if (input_tokens > (1LL << 40) || output_tokens > (1LL << 31)) return fail(h, RSIM_E_TRACE, "request: token count too large");
    if (n_holders < 0 || (n_holders > 0 && !holders)) return fail(h, RSIM_E_INVALID, "bad holders");
    CK(h, cudaSetDevice(h->cfg.device));
    const int N = h->cfg.n_instances;
    const i64 words = n_holders > 0 ? ((i64)N + 31) / 32 : 0;
    const size_t need = RQ_HDR + (size_t)words + (size_t)n_blocks;
    cudaStream_t st = h->stream;
    if (need > h->rq_cap) {
        if (h->rq_h) { CK(h, cudaStreamSynchronize(st)); CK(h, cudaFreeHost(h->rq_h)); h->rq_h = nullptr; }
        const size_t cap = std::max<size_t>(need * 2, 4096);
        void *p = nullptr;
        CK(h, cudaHostAlloc(&p, cap * sizeof(i64), cudaHostAllocDefault));
        h->rq_h = (i64 *)p; h->rq_cap = cap;
        CK(h, h->rq_dev.reserve(cap, 0, st));
    }
    if (!h->ro_h) {
        void *p = nullptr;
        // decision, error word, flag + up to 5N + 1 scores (the detector's route() layout) + diagnostics
        CK(h, cudaHostAlloc(&p, (RO_HDR + 5 * (size_t)h->N + 16) * sizeof(i64), cudaHostAllocMapped));
        h->ro_h = (i64 *)p;
        CK(h, cudaHostGetDevicePointer((void **)&h->ro_d, p, 0));
    }
    const i64 bs = h->cfg.block_size;
    const i64 R0 = h->R, R1 = R0 + 1, no = (output_tokens + bs - 1) / bs;
    CK(h, h->arrival.reserve(R1, R0, st)); CK(h, h->in_tok.reserve(R1, R0, st)); CK(h, h->out_tok.reserve(R1, R0, st));
    CK(h, h->rid.reserve(R1, R0, st)); CK(h, h->blk_off.reserve(R1 + 1, R0 + 1, st)); CK(h, h->ooff.reserve(R1 + 1, R0 + 1, st));
    CK(h, h->blocks.reserve(h->nblk + n_blocks, h->nblk, st)); CK(h, h->ckeys.reserve(h->nblk + n_blocks, h->nblk, st));
    CK(h, h->okeys.reserve(h->nout + no + 1, h->nout, st));
    CK(h, h->hit_blocks.reserve(R1, R0, st)); CK(h, h->chosen.reserve(R1, R0, st));
    DevArr<i64> *outs[] = {&h->hit_tokens, &h->first_sched, &h->first_token, &h->finish, &h->route_bs, &h->dec_ns};
    for (auto *a : outs) CK(h, a->reserve(R1, R0, st));
    if (words) CK(h, h->dupmask.reserve(words, 0, st));
    int trk = -1, newt = -1;
    if (h->cfg.det_on) {                      // the request's class (rsim_detector_next)
        trk = h->det_next_track;
        const int T0 = h->det_loaded ? h->dT : 0;
        newt = trk == T0 ? trk : -1;
        rsim_status ds = det_ensure(h, std::max(T0, trk + 1), R1, h->det_next_rows);
        if (ds != RSIM_OK) return ds;
        h->det_next_track = -1;
    }
    i64 *q = h->rq_h;
    q[RQ_ARRIVAL] = now_us; q[RQ_IN] = input_tokens; q[RQ_OUT] = output_tokens; q[RQ_RID] = (i64)request_id;
    q[RQ_B] = n_blocks; q[RQ_R0] = R0; q[RQ_NBLK0] = h->nblk; q[RQ_NOUT0] = h->nout; q[RQ_NO] = no; q[RQ_NDUP] = words;
    q[RQ_TRACK] = trk; q[RQ_NEWT] = newt; q[RQ_EXLEN] = h->det_next_len; q[RQ_CKEY] = (i64)h->det_next_key;
    for (i64 w = 0; w < words; w++) q[RQ_HDR + w] = 0;
    for (int i = 0; i < n_holders; i++) {
        if (holders[i] < 0 || holders[i] >= N) return fail(h, RSIM_E_INVALID, "holder out of range");
        q[RQ_HDR + (holders[i] >> 5)] |= (i64)(1u << (holders[i] & 31));
    }
    memcpy(q + RQ_HDR + words, blocks, (size_t)n_blocks * sizeof(u64));
    CK(h, cudaMemcpyAsync(h->rq_dev.p, q, need * sizeof(i64), cudaMemcpyHostToDevice, st));
    const bool filt = h->cfg.policy == RSIM_POLICY_FILTER;
    const int nsc = h->cfg.det_on ? 5 * h->N + 1 : (filt ? 2 : 1) * h->N;
    rsim_status rs = RSIM_OK;
    if (h->route1) {
        // plain policies on one rank with <= 1024 instances: the whole call is one launch
        Params P = make_params(h);
        P.scores = h->scores;
        P.dupmask = nullptr;                      // (route_kernel reads the holders from the request block)
        const int nw = std::min(RK_MAXW, h->N);         // instances spread over up to 32 warps
        // (results straight to mapped memory: a device block + D2H copy measured 7-10 us slower)
        route_kernel<<<1, 32 * nw, (size_t)nw * sizeof(WarpBuf) + (size_t)h->N * sizeof(Inst), st>>>(
            P, h->rq_dev.p, h->ro_d, nsc, h->blocks.p);
        h->launches++;
        CK(h, cudaGetLastError());
        if (R0 > 0 && now_us < h->last_arrival) h->order_breaks.push_back(R0);
        h->last_arrival = now_us;
        h->R = R1; h->nblk += n_blocks; h->nout += no;
    } else {
    route_ingest_kernel<<<1, 32, 0, st>>>(h->rq_dev.p, h->arrival.p, h->in_tok.p, h->out_tok.p, h->rid.p, h->blk_off.p,
                                          h->ooff.p, h->blocks.p, h->ckeys.p, h->okeys.p, h->chosen.p, h->hit_blocks.p,
                                          h->hit_tokens.p, h->first_sched.p, h->first_token.p, h->finish.p,
                                          h->route_bs.p, h->dec_ns.p, h->dupmask.p, h->flag,
                                          h->cfg.det_on ? h->dtid.p : nullptr, h->dtw.p, h->dtex.p, h->dtkey.p);
    h->launches++;
    CK(h, cudaGetLastError());
    if (R0 > 0 && now_us < h->last_arrival) h->order_breaks.push_back(R0);
    h->last_arrival = now_us;
    h->R = R1; h->nblk += n_blocks; h->nout += no;
    h->cur_dupmask = words ? h->dupmask.p : nullptr;
    rs = launch_replay(h, R0, R1, now_us, MODE_ROUTE, -1, h->scores, nullptr, false);
    h->cur_dupmask = nullptr;
    if (rs != RSIM_OK) { cudaStreamSynchronize(st); return rs; }
    route_out_kernel<<<1, 128, 0, st>>>(h->chosen.p, h->hit_tokens.p, R0, h->scores, nsc, h->errbuf, h->flag, h->ro_d);
    h->launches++;
    CK(h, cudaGetLastError());
    }
    CK(h, cudaStreamSynchronize(st));
    const i64 *o = h->ro_h;
#ifdef RSIM_ROUTE_TIMING
    if (h->route1) {            // diagnostics: route_kernel phase times (ns), averaged at destroy
        static double acc[8] = {0};
        static long calls = 0;
        for (int i = 0; i < 7; i++) acc[i] += (double)(o[RO_HDR + nsc + i + 1] - o[RO_HDR + nsc + i]);
        if (++calls % 1000 == 0) {
            fprintf(stderr, "[route_kernel ns/phase over %ld calls] ingest %.0f load %.0f probe+score %.0f "
                    "warpmin %.0f decide %.0f commit %.0f tail %.0f\n", calls, acc[0] / calls, acc[1] / calls,
                    acc[2] / calls, acc[3] / calls, acc[4] / calls, acc[5] / calls, acc[6] / calls);
        }
    }
#endif
    const int e[4] = {(int)o[RO_ERR0], (int)o[RO_ERR1], (int)o[RO_ERR2], (int)o[RO_ERR3]};
    if ((rs = decode_device_error(h, e)) != RSIM_OK) {
        // a refused duplicate never reaches Detector.observe (cluster.py:140-142): a track it
        // opened was not created, and the next new class takes its slot
        if (rs == RSIM_E_DUPLICATE && newt >= 0) h->dT = newt;
        return rs;
    }
    if (o[RO_FLAG]) return fail(h, RSIM_E_TRACE, "a chain key equals the table sentinel 0 (probability 2^-64 per key)");
    if (chosen) *chosen = (int32_t)o[RO_CHOSEN];
    if (hit_tokens) *hit_tokens = o[RO_HIT];
    const double *sc = reinterpret_cast<const double *>(o + RO_HDR);
    // the detector's verdict (policies.py:222-236): 0 none (or fail open), 2 holders excluded,
    // 3 forced least_bs, 4 holders excluded and route_filter's batch-size branch over the rest
    const int code = h->cfg.det_on ? (int)sc[5 * N] : 0;
    if (branch) *branch = code;
    if (scores) {
        const double *pick = sc;
        if (code == 3) {
            pick = sc + 2 * N;                                  // least_bs: float(bs)
        } else if (code == 2 || code == 4) {                    // the kept candidates only (NaN: excluded)
            const double *base = code == 4 ? sc + N
                               : (h->cfg.policy == RSIM_POLICY_LINEAR && !(h->cfg.bs_norm_cap > 0)) ? sc + 4 * N : sc;
            for (int i = 0; i < N; i++) scores[i] = sc[3 * N + i] != 0.0 ? std::nan("") : base[i];
            return RSIM_OK;
        } else if (filt) {       // the branch route_filter took (policies.py:180-183)
            const auto mm = std::minmax_element(sc + N, sc + 2 * N);
            if ((i64)*mm.second - (i64)*mm.first > h->cfg.range_threshold) pick = sc + N;
        }
        memcpy(scores, pick, N * sizeof(double));
    }
    return RSIM_OK;
}

// InstanceSim.queue / .running of one local instance (engine.py:212-213): 8 int64 per slot, the
// FIFO queue in order, then the running list in order: request index, kind (0 queued, 1 running),
// pending prefill tokens, generated tokens, hit blocks, input tokens, output tokens, flags.
rsim_status rsim_read_slots(rsim_t *h, int32_t instance, int64_t *out, int64_t cap, int64_t *n_queued,
                            int64_t *n_running) {
    if (!h) return RSIM_E_INVALID;
    if (instance < 0 || instance >= h->N) return fail(h, RSIM_E_INVALID, "instance out of range");
    CK(h, cudaSetDevice(h->cfg.device));
    CK(h, cudaStreamSynchronize(h->stream));
    Inst s;
    CK(h, cudaMemcpy(&s, h->inst + instance, sizeof(Inst), cudaMemcpyDeviceToHost));
    if (n_queued) *n_queued = s.q;
    if (n_running) *n_running = s.r;
    if (!out) return RSIM_OK;
    if (cap < (i64)s.q + s.r) return fail(h, RSIM_E_INVALID, "slot buffer too small (%d needed)", s.q + s.r);
    const int qcap = 1 << h->qlog2;
    std::vector<Ent> ring(qcap), run(std::max(s.r, 1));
    CK(h, cudaMemcpy(ring.data(), h->qbuf + ((size_t)instance << h->qlog2), qcap * sizeof(Ent), cudaMemcpyDeviceToHost));
    if (s.r) CK(h, cudaMemcpy(run.data(), h->rbuf + (size_t)instance * h->cfg.max_batch_requests, s.r * sizeof(Ent),
                              cudaMemcpyDeviceToHost));
    int64_t *o = out;
    for (int j = 0; j < s.q; j++, o += 8) {
        const Ent &e = ring[(s.q_head + j) & (qcap - 1)];
        o[0] = e.req; o[1] = 0; o[2] = e.v; o[3] = 0; o[4] = e.hb; o[5] = e.in; o[6] = e.out; o[7] = e.flags;
    }
    for (int j = 0; j < s.r; j++, o += 8) {      // finish step v = join step + out - 1
        const Ent &e = run[j];
        o[0] = e.req; o[1] = 1; o[2] = 0; o[3] = (i64)e.out - 1 - (e.v - s.step_idx); o[4] = e.hb; o[5] = e.in;
        o[6] = e.out; o[7] = e.flags;
    }
    return RSIM_OK;
}

// run_trace's loops start with no step scheduled (cluster.py:210-211, 247): route()/enqueue() API
// calls before it leave their instances idle-but-queued until an arrival is routed there.
rsim_status rsim_unschedule(rsim_t *h) {
    if (!h) return RSIM_E_INVALID;
    CK(h, cudaSetDevice(h->cfg.device));
    CK(h, cudaStreamSynchronize(h->stream));
    std::vector<Inst> hs(h->N);
    CK(h, cudaMemcpy(hs.data(), h->inst, h->N * sizeof(Inst), cudaMemcpyDeviceToHost));
    for (auto &s : hs) s.next_step = RSIM_NONE;
    CK(h, cudaMemcpy(h->inst, hs.data(), h->N * sizeof(Inst), cudaMemcpyHostToDevice));
    return RSIM_OK;
}

rsim_status rsim_enqueue(rsim_t *h, int32_t instance, int64_t r, int64_t now_us, int64_t *hit_tokens) {
    if (!h) return RSIM_E_INVALID;
    if (r < 0 || r >= h->R) return fail(h, RSIM_E_INVALID, "request index out of range");
    if (instance < 0 || instance >= h->N) return fail(h, RSIM_E_INVALID, "instance out of range");
    CK(h, cudaSetDevice(h->cfg.device));
    rsim_status st = launch_replay(h, r, r + 1, now_us, MODE_ENQUEUE, instance, nullptr, nullptr);
    if (st != RSIM_OK) return st;
    if (hit_tokens) CK(h, cudaMemcpy(hit_tokens, h->hit_tokens.p + r, sizeof(i64), cudaMemcpyDeviceToHost));
    return RSIM_OK;
}

static rsim_status arena_append(rsim_t *h, const uint64_t *keys, int64_t n, i64 *a0) {
    CK(h, h->arena.reserve(h->narena + n + 1, h->narena, h->stream));
    if (n) CK(h, cudaMemcpy(h->arena.p + h->narena, keys, n * sizeof(u64), cudaMemcpyHostToDevice));
    *a0 = h->narena;
    h->narena += n;
    return RSIM_OK;
}

rsim_status rsim_cache_insert_keys(rsim_t *h, int32_t instance, const uint64_t *keys, int64_t n, int64_t now_us,
                                   int64_t *evicted) {
    if (!h) return RSIM_E_INVALID;
    if (instance < 0 || instance >= h->N) return fail(h, RSIM_E_INVALID, "instance out of range");
    for (i64 i = 0; i < n; i++) if (keys[i] == 0) return fail(h, RSIM_E_INVALID, "key equals the table sentinel 0");
    CK(h, cudaSetDevice(h->cfg.device));
    i64 a0 = 0;
    rsim_status st = arena_append(h, keys, n, &a0);
    if (st) return st;
    h->api_segs.insert(h->api_segs.end(), {(i64)instance, a0, (i64)n});
    cache_op_kernel<<<1, 32, 0, h->stream>>>(make_params(h), instance, 0, a0, (int)n, now_us, h->scratch_res);
    h->launches++;
    CK(h, cudaGetLastError());
    i64 res = 0;
    CK(h, cudaMemcpyAsync(&res, h->scratch_res, sizeof(i64), cudaMemcpyDeviceToHost, h->stream));
    st = check_device_error(h);
    if (st) return st;
    if (evicted) *evicted = res;
    return RSIM_OK;
}

rsim_status rsim_cache_match_keys(rsim_t *h, int32_t instance, const uint64_t *keys, int64_t n, int64_t *hit) {
    if (!h) return RSIM_E_INVALID;
    if (instance < 0 || instance >= h->N) return fail(h, RSIM_E_INVALID, "instance out of range");
    CK(h, cudaSetDevice(h->cfg.device));
    i64 a0 = 0;
    rsim_status st = arena_append(h, keys, n, &a0);     // (match keys are not named by runs; reuse the slot)
    if (st) return st;
    h->narena = a0;
    cache_op_kernel<<<1, 32, 0, h->stream>>>(make_params(h), instance, 1, a0, (int)n, 0, h->scratch_res);
    h->launches++;
    CK(h, cudaGetLastError());
    i64 res = 0;
    CK(h, cudaMemcpyAsync(&res, h->scratch_res, sizeof(i64), cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    if (hit) *hit = res;
    return RSIM_OK;
}

rsim_status rsim_probe_batch(rsim_t *h, int64_t first, int64_t count, int32_t *out) {
    if (!h) return RSIM_E_INVALID;
    if (first < 0 || count < 0 || first + count > h->R) return fail(h, RSIM_E_INVALID, "request range out of the loaded trace");
    CK(h, cudaSetDevice(h->cfg.device));
    int *d = nullptr;
    const size_t n = (size_t)count * h->N;
    CK(h, cudaMalloc(&d, std::max<size_t>(n, 1) * sizeof(int)));
    CK(h, cudaEventRecord(h->ev0, h->stream));
    {   // a thread per (request, instance) pair, grid-stride, 8 resident blocks per SM
        const int grid = (int)std::min<i64>(((i64)n + 255) / 256, 148 * 8);
        static const int depth = getenv("RSIM_PROBE_DEPTH") ? atoi(getenv("RSIM_PROBE_DEPTH")) : 3;   // A/B switch (D = 2 / 3 / 4: api64 0.194 / 0.189 / 0.188 ms, chat1024 1.32 / 1.34 / 1.38, agent256 4.16 / 3.88 / 3.68)
        if (depth >= 4) probe_scan_kernel<4><<<std::max(grid, 1), 256, 0, h->stream>>>(make_params(h), first, count, d);
        else if (depth == 3) probe_scan_kernel<3><<<std::max(grid, 1), 256, 0, h->stream>>>(make_params(h), first, count, d);
        else probe_scan_kernel<2><<<std::max(grid, 1), 256, 0, h->stream>>>(make_params(h), first, count, d);
    }
    h->launches++;
    CK(h, cudaGetLastError());
    CK(h, cudaEventRecord(h->ev1, h->stream));
    CK(h, cudaMemcpyAsync(out, d, n * sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    cudaEventElapsedTime(&h->last_replay_ms, h->ev0, h->ev1);
    cudaFree(d);
    return RSIM_OK;
}

rsim_status rsim_chain_keys(rsim_t *h, const uint64_t *blocks, int64_t n, uint64_t *keys_out) {
    if (!h) return RSIM_E_INVALID;
    if (n <= 0) return RSIM_OK;
    CK(h, cudaSetDevice(h->cfg.device));
    u64 *db = nullptr, *dk = nullptr, *dok = nullptr, *drid = nullptr;
    i64 *doff = nullptr, *doo = nullptr;
    int *dflag = nullptr;
    i64 off[2] = {0, n}, oo[2] = {0, 0};
    u64 rid0 = 0;
    CK(h, cudaMalloc(&db, n * sizeof(u64))); CK(h, cudaMalloc(&dk, n * sizeof(u64)));
    CK(h, cudaMalloc(&dok, sizeof(u64))); CK(h, cudaMalloc(&drid, sizeof(u64)));
    CK(h, cudaMalloc(&doff, 2 * sizeof(i64))); CK(h, cudaMalloc(&doo, 2 * sizeof(i64)));
    CK(h, cudaMalloc(&dflag, sizeof(int)));
    CK(h, cudaMemcpy(db, blocks, n * sizeof(u64), cudaMemcpyHostToDevice));
    CK(h, cudaMemcpy(doff, off, sizeof(off), cudaMemcpyHostToDevice));
    CK(h, cudaMemcpy(doo, oo, sizeof(oo), cudaMemcpyHostToDevice));
    CK(h, cudaMemcpy(drid, &rid0, sizeof(u64), cudaMemcpyHostToDevice));
    k1_chain_keys<<<1, 32 * K1_WARPS, 0, h->stream>>>(doff, db, dk, doo, dok, drid, 0, 1, 0ULL, dflag);
    h->launches++;
    CK(h, cudaGetLastError());
    CK(h, cudaStreamSynchronize(h->stream));
    CK(h, cudaMemcpy(keys_out, dk, n * sizeof(u64), cudaMemcpyDeviceToHost));
    cudaFree(db); cudaFree(dk); cudaFree(dok); cudaFree(drid); cudaFree(doff); cudaFree(doo); cudaFree(dflag);
    return RSIM_OK;
}

static rsim_status read_range(rsim_t *h, void *dst, const void *src, size_t elem, i64 first, i64 count) {
    if (!dst || count == 0) return RSIM_OK;
    if (first < 0 || count < 0 || first + count > h->R) return fail(h, RSIM_E_INVALID, "range out of the loaded trace");
    CK(h, cudaMemcpy(dst, (const char *)src + first * elem, count * elem, cudaMemcpyDeviceToHost));
    return RSIM_OK;
}

rsim_status rsim_read_decisions(rsim_t *h, int64_t first, int64_t count, int32_t *chosen, int64_t *hit) {
    if (!h) return RSIM_E_INVALID;
    CK(h, cudaSetDevice(h->cfg.device));
    rsim_status st = read_range(h, chosen, h->chosen.p, sizeof(int), first, count);
    if (st) return st;
    return read_range(h, hit, h->hit_tokens.p, sizeof(i64), first, count);
}

rsim_status rsim_read_request_times(rsim_t *h, int64_t first, int64_t count, int64_t *fs, int64_t *ft, int64_t *fin) {
    if (!h) return RSIM_E_INVALID;
    CK(h, cudaSetDevice(h->cfg.device));
    rsim_status st = read_range(h, fs, h->first_sched.p, sizeof(i64), first, count);
    if (st) return st;
    st = read_range(h, ft, h->first_token.p, sizeof(i64), first, count);
    if (st) return st;
    return read_range(h, fin, h->finish.p, sizeof(i64), first, count);
}

rsim_status rsim_read_route_bs(rsim_t *h, int64_t first, int64_t count, int64_t *bs) {
    if (!h) return RSIM_E_INVALID;
    CK(h, cudaSetDevice(h->cfg.device));
    return read_range(h, bs, h->route_bs.p, sizeof(i64), first, count);
}

rsim_status rsim_read_decision_ns(rsim_t *h, int64_t first, int64_t count, int64_t *ns) {
    if (!h) return RSIM_E_INVALID;
    CK(h, cudaSetDevice(h->cfg.device));
    return read_range(h, ns, h->dec_ns.p, sizeof(i64), first, count);
}

rsim_status rsim_read_instances(rsim_t *h, int64_t *out) {
    if (!h || !out) return RSIM_E_INVALID;
    CK(h, cudaSetDevice(h->cfg.device));
    const int N = h->N;
    std::vector<Inst> hs(N);
    CK(h, cudaMemcpy(hs.data(), h->inst, N * sizeof(Inst), cudaMemcpyDeviceToHost));
    for (int i = 0; i < N; i++) {
        const Inst &s = hs[i];
        int64_t *o = out + 12 * i;
        o[0] = s.r; o[1] = s.q; o[2] = s.pend; o[3] = s.total; o[4] = s.dcs;
        o[5] = s.v_r; o[6] = s.v_q; o[7] = s.v_pend; o[8] = s.v_total; o[9] = s.v_dc;
        o[10] = s.busy_until; o[11] = s.occ;
    }
    return RSIM_OK;
}

rsim_status rsim_read_step_log(rsim_t *h, int64_t *out, int64_t cap, int64_t *n_records) {
    if (!h) return RSIM_E_INVALID;
    CK(h, cudaSetDevice(h->cfg.device));
    u64 n = 0;
    CK(h, cudaMemcpy(&n, h->log_n, sizeof(u64), cudaMemcpyDeviceToHost));
    if (n_records) *n_records = (i64)n;
    if (!h->log) return fail(h, RSIM_E_INVALID, "step log disabled (record_steps = 0)");
    if ((i64)n > h->log_cap) return fail(h, RSIM_E_INVALID, "step log overflowed its capacity (%lld)", (long long)h->log_cap);
    if ((i64)n > cap) return fail(h, RSIM_E_INVALID, "output buffer too small");
    // through a pinned bounce buffer, double-buffered (the DMA of chunk c+1 runs while chunk c is
    // compacted into out); records are reserved per warp in chunks (log_step): drop the unused
    // ones (gi = -1)
    const i64 CH = 1 << 17;                                   // records per chunk (6 MB)
    if (!h->log_pin) {
        void *p = nullptr;
        CK(h, cudaHostAlloc(&p, 2 * CH * 6 * sizeof(i64), cudaHostAllocDefault));
        h->log_pin = (i64 *)p;
    }
    i64 m = 0;
    const i64 nc = ((i64)n + CH - 1) / CH;
    if (nc) CK(h, cudaMemcpyAsync(h->log_pin, h->log, std::min<i64>(CH, n) * 6 * sizeof(i64), cudaMemcpyDeviceToHost, h->stream));
    for (i64 c = 0; c < nc; c++) {
        CK(h, cudaStreamSynchronize(h->stream));
        if (c + 1 < nc) {
            const i64 o = (c + 1) * CH, len = std::min<i64>(CH, (i64)n - o);
            CK(h, cudaMemcpyAsync(h->log_pin + ((c + 1) & 1) * CH * 6, h->log + o * 6, len * 6 * sizeof(i64),
                                  cudaMemcpyDeviceToHost, h->stream));
        }
        const i64 *src = h->log_pin + (c & 1) * CH * 6;
        const i64 len = std::min<i64>(CH, (i64)n - c * CH);
        for (i64 i = 0; i < len; i++)
            if (src[6 * i] >= 0) { memcpy(out + 6 * m, src + 6 * i, 6 * sizeof(i64)); m++; }
    }
    if (n_records) *n_records = m;
    return RSIM_OK;
}

// Whole-trace replay on the resident trace: reset engine/KV$/tie state, rerun
// K1 over the loaded trace, replay every decision, drain to idle. The device
// time of that sequence (CUDA events on the handle's stream) -> *device_ms.
rsim_status rsim_rerun(rsim_t *h, double *device_ms) {
    if (!h) return RSIM_E_INVALID;
    CK(h, cudaSetDevice(h->cfg.device));
    cudaStream_t s = h->stream;
    const int N = h->N;
    h->epoch += 1;
    std::vector<Inst> hs(N);
    for (auto &x : hs) x = fresh_inst();
    u64 tie[2] = {h->cfg.tie_seed_lo, h->cfg.tie_seed_hi};
    cudaEvent_t e0, e1, ek0, ek1;
    CK(h, cudaEventCreate(&e0));
    CK(h, cudaEventCreate(&e1));
    CK(h, cudaEventCreate(&ek0));
    CK(h, cudaEventCreate(&ek1));
    CK(h, cudaEventRecord(e0, s));
    const size_t slots = (size_t)N << h->slog2;
    CK(h, cudaMemcpyAsync(h->inst, hs.data(), N * sizeof(Inst), cudaMemcpyHostToDevice, s));
    if (det_reset(h, s) != RSIM_OK) return RSIM_E_CUDA;
    CK(h, cudaMemsetAsync(h->tkeys, 0, slots * sizeof(u64), s));
    CK(h, cudaMemsetAsync(h->tmeta, 0, slots * sizeof(Meta), s));
    CK(h, cudaMemcpyAsync(h->tie, tie, sizeof(tie), cudaMemcpyHostToDevice, s));
    CK(h, cudaMemsetAsync(h->log_n, 0, sizeof(u64), s));
    CK(h, cudaMemsetAsync(h->ctr, 0, 48 * sizeof(u64), s));
    if (h->R > 0) {
        DevArr<i64> *outs[] = {&h->hit_tokens, &h->first_sched, &h->first_token, &h->finish, &h->route_bs, &h->dec_ns};
        for (auto *a : outs) CK(h, cudaMemsetAsync(a->p, 0xff, h->R * sizeof(i64), s));
        CK(h, cudaMemsetAsync(h->chosen.p, 0xff, h->R * sizeof(int), s));
        const i64 nwarps = (h->R + 31) / 32;
        CK(h, cudaEventRecord(ek0, s));                     // K1 alone (rsim_last_timings' k1_ms)
        k1_chain_keys<<<(int)((nwarps + K1_WARPS - 1) / K1_WARPS), 32 * K1_WARPS, 0, s>>>(
            h->blk_off.p, h->blocks.p, h->ckeys.p, h->ooff.p, h->okeys.p, h->rid.p, 0, h->R, 0ULL, h->flag);
        h->launches++;
        CK(h, cudaGetLastError());
        CK(h, cudaEventRecord(ek1, s));
        rsim_status st = launch_replay(h, 0, h->R, 0, MODE_REPLAY, -1, nullptr, &h->last_replay_ms);
        if (st != RSIM_OK) { cudaEventDestroy(e0); cudaEventDestroy(e1); cudaEventDestroy(ek0); cudaEventDestroy(ek1); return st; }
        cudaEventElapsedTime(&h->last_k1_ms, ek0, ek1);     // (launch_replay synchronised the stream)
    }
    rsim_status st = launch_replay(h, 0, 0, RSIM_NONE, MODE_DRAIN, -1, nullptr, &h->last_drain_ms);
    CK(h, cudaEventRecord(e1, s));
    CK(h, cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (device_ms) *device_ms = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(ek0);
    cudaEventDestroy(ek1);
    return st;
}

rsim_status rsim_read_counters(rsim_t *h, int64_t *out16) {
    if (!h || !out16) return RSIM_E_INVALID;
    CK(h, cudaSetDevice(h->cfg.device));
    u64 c[16];
    CK(h, cudaMemcpy(c, h->ctr, sizeof(c), cudaMemcpyDeviceToHost));
    for (int i = 0; i < 16; i++) out16[i] = (int64_t)c[i];
    out16[4] = h->R; out16[5] = h->nblk; out16[7] = h->N;
    return RSIM_OK;
}

rsim_status rsim_read_step_cycles(rsim_t *h, int64_t *out32) {
    if (!h || !out32) return RSIM_E_INVALID;
    CK(h, cudaSetDevice(h->cfg.device));
    u64 c[32];
    CK(h, cudaMemcpy(c, h->ctr + 16, sizeof(c), cudaMemcpyDeviceToHost));
    for (int i = 0; i < 32; i++) out32[i] = (int64_t)c[i];
    return RSIM_OK;
}

rsim_status rsim_phase_records(rsim_t *h, int64_t capacity_decisions) {
    if (!h || capacity_decisions < 0) return RSIM_E_INVALID;
    CK(h, cudaSetDevice(h->cfg.device));
    if (h->crit) { cudaFree(h->crit); h->crit = nullptr; }
    h->crit_cap = 0;
    if (capacity_decisions == 0) return RSIM_OK;
    // records [n][C*W][8] u16, then the timeline [n][C*W + 4] u64 (%globaltimer)
    const size_t bytes = (size_t)capacity_decisions * h->C * h->W * 8 * sizeof(unsigned short) +
                         (size_t)capacity_decisions * (h->C * h->W + 4) * sizeof(u64);
    CK(h, cudaMalloc(&h->crit, bytes));
    CK(h, cudaMemset(h->crit, 0, bytes));
    h->crit_cap = capacity_decisions;
    return RSIM_OK;
}

rsim_status rsim_read_phase_records(rsim_t *h, uint16_t *out, int64_t n_decisions, int32_t *warps_per_decision) {
    if (!h) return RSIM_E_INVALID;
    if (warps_per_decision) *warps_per_decision = h->C * h->W;
    if (!out || n_decisions <= 0) return RSIM_OK;
    if (n_decisions > h->crit_cap) return fail(h, RSIM_E_INVALID, "more decisions than recorded");
    CK(h, cudaSetDevice(h->cfg.device));
    CK(h, cudaMemcpy(out, h->crit, (size_t)n_decisions * h->C * h->W * 8 * sizeof(unsigned short),
                     cudaMemcpyDeviceToHost));
    return RSIM_OK;
}

rsim_status rsim_read_phase_times(rsim_t *h, uint64_t *out, int64_t n_decisions) {
    if (!h || !out) return RSIM_E_INVALID;
    if (n_decisions > h->crit_cap) return fail(h, RSIM_E_INVALID, "more decisions than recorded");
    CK(h, cudaSetDevice(h->cfg.device));
    const size_t off = (size_t)h->crit_cap * h->C * h->W * 8;
    CK(h, cudaMemcpy(out, h->crit + off, (size_t)n_decisions * (h->C * h->W + 4) * sizeof(u64),
                     cudaMemcpyDeviceToHost));
    return RSIM_OK;
}

rsim_status rsim_shard_bounds(const rsim_t *h, int32_t *lo, int32_t *hi) {
    if (!h) return RSIM_E_INVALID;
    if (lo) *lo = h->gbase;
    if (hi) *hi = h->gbase + h->N;
    return RSIM_OK;
}

rsim_status rsim_mailbox(rsim_t *h, void **dev_ptr) {
    if (!h || !dev_ptr) return RSIM_E_INVALID;
    *dev_ptr = h->mbox;
    return RSIM_OK;
}

rsim_status rsim_mailbox_ipc_handle(rsim_t *h, unsigned char out64[64]) {
    if (!h || !out64) return RSIM_E_INVALID;
    CK(h, cudaSetDevice(h->cfg.device));
    cudaIpcMemHandle_t ih;
    CK(h, cudaIpcGetMemHandle(&ih, h->mbox));
    memcpy(out64, &ih, 64);
    return RSIM_OK;
}

rsim_status rsim_set_peer(rsim_t *h, int32_t rank, void *peer_mailbox) {
    if (!h || rank < 0 || rank >= 8 || !peer_mailbox) return RSIM_E_INVALID;
    h->peer[rank] = (u64 *)peer_mailbox;
    return RSIM_OK;
}

rsim_status rsim_open_peer_ipc(rsim_t *h, int32_t rank, const unsigned char in64[64]) {
    if (!h || rank < 0 || rank >= 8 || !in64) return RSIM_E_INVALID;
    CK(h, cudaSetDevice(h->cfg.device));
    cudaIpcMemHandle_t ih;
    memcpy(&ih, in64, 64);
    void *p = nullptr;
    CK(h, cudaIpcOpenMemHandle(&p, ih, cudaIpcMemLazyEnablePeerAccess));
    h->peer[rank] = (u64 *)p;
    h->peer_ipc[rank] = true;
    return RSIM_OK;
}

rsim_status rsim_last_timings(rsim_t *h, double *replay_ms, double *k1_ms, double *drain_ms) {
    if (!h) return RSIM_E_INVALID;
    if (replay_ms) *replay_ms = h->last_replay_ms;
    if (k1_ms) *k1_ms = h->last_k1_ms;
    if (drain_ms) *drain_ms = h->last_drain_ms;
    return RSIM_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- hotspot detector
rsim_status rsim_load_detector(rsim_t *h, int64_t n, const int32_t *track_of_request, int32_t n_tracks,
                               const int64_t *exemplar_offset, const int32_t *exemplar_len, const uint64_t *class_key,
                               int64_t rows_capacity) {
    if (!h) return RSIM_E_INVALID;
    if (!h->cfg.det_on) return fail(h, RSIM_E_INVALID, "handle was created without a detector");
    if (n != h->R || h->R == 0) return fail(h, RSIM_E_INVALID, "rsim_load_detector needs the loaded trace (%lld requests)", (long long)h->R);
    if (n_tracks < 1 || !track_of_request || !exemplar_offset || !exemplar_len || !class_key)
        return fail(h, RSIM_E_INVALID, "null / empty detector classes");
    int next = 0;
    for (i64 r = 0; r < n; r++) {                  // dense ids by first arrival
        if (track_of_request[r] < 0 || track_of_request[r] > next || track_of_request[r] >= n_tracks)
            return fail(h, RSIM_E_INVALID, "track ids must be numbered by first arrival");
        if (track_of_request[r] == next) next++;
    }
    if (next != n_tracks) return fail(h, RSIM_E_INVALID, "unused detector tracks");
    for (int t = 0; t < n_tracks; t++)
        if (exemplar_len[t] < 1 || exemplar_offset[t] < 0 || exemplar_offset[t] + exemplar_len[t] > h->nblk)
            return fail(h, RSIM_E_INVALID, "bad exemplar of track %d", t);
    CK(h, cudaSetDevice(h->cfg.device));
    cudaStream_t s = h->stream;
    const int T = n_tracks;
    int bl = 0;
    while ((1LL << bl) < (i64)h->cfg.det_window_s + 2) bl++;
    CK(h, h->dtid.reserve(n, 0, s)); CK(h, h->dtw.reserve(T, 0, s)); CK(h, h->dtex.reserve(T, 0, s));
    CK(h, h->dtkey.reserve(T, 0, s)); CK(h, h->dtr.reserve(T, 0, s));
    CK(h, h->dbk.reserve(((size_t)T * 3 << bl) * h->C, 0, s));   // one bucket ring set per CTA
    const i64 rc = std::max<i64>(rows_capacity, 16);
    CK(h, h->drows.reserve((size_t)rc * 7, 0, s));
    if (!h->dtot || bl > h->dbclog2) {
        if (h->dtot) cudaFree(h->dtot);
        CK(h, cudaMalloc(&h->dtot, ((size_t)2 << bl) * h->C * sizeof(i64)));
    }
    if (!h->dglob) CK(h, cudaMalloc(&h->dglob, DG_N * sizeof(i64)));
    CK(h, cudaMemcpyAsync(h->dtid.p, track_of_request, n * sizeof(int), cudaMemcpyHostToDevice, s));
    CK(h, cudaMemcpyAsync(h->dtw.p, exemplar_len, T * sizeof(int), cudaMemcpyHostToDevice, s));
    CK(h, cudaMemcpyAsync(h->dtex.p, exemplar_offset, T * sizeof(i64), cudaMemcpyHostToDevice, s));
    CK(h, cudaMemcpyAsync(h->dtkey.p, class_key, T * sizeof(u64), cudaMemcpyHostToDevice, s));
    h->dT = T; h->dTs = T; h->dbclog2 = bl; h->drows_cap = rc;
    if (getenv("RSIM_DET_DEBUG")) {
        CK(h, h->ddbg.reserve((size_t)n * (8 + h->N), 0, s));
        CK(h, cudaMemsetAsync(h->ddbg.p, 0xff, (size_t)n * (8 + h->N) * sizeof(i64), s));
    }
    h->det_loaded = true;
    return det_reset(h, s);
}

rsim_status rsim_detector_finalize(rsim_t *h) {
    if (!h) return RSIM_E_INVALID;
    if (!h->cfg.det_on || !h->det_loaded) return fail(h, RSIM_E_INVALID, "no detector classes loaded");
    CK(h, cudaSetDevice(h->cfg.device));
    det_finalize_kernel<<<1, 32, 0, h->stream>>>(make_params(h));
    CK(h, cudaGetLastError());
    h->launches += 1;
    CK(h, cudaStreamSynchronize(h->stream));
    return check_device_error(h);
}

rsim_status rsim_read_detector(rsim_t *h, int64_t *rows, int64_t capacity, int64_t *n_rows, int64_t *first_violation_us) {
    if (!h) return RSIM_E_INVALID;
    if (!h->cfg.det_on || !h->det_loaded) return fail(h, RSIM_E_INVALID, "no detector classes loaded");
    CK(h, cudaSetDevice(h->cfg.device));
    i64 g[DG_N];
    CK(h, cudaMemcpy(g, h->dglob, sizeof(g), cudaMemcpyDeviceToHost));
    if (n_rows) *n_rows = g[DG_NROWS];
    if (first_violation_us) *first_violation_us = g[DG_FIRSTV];
    const i64 m = std::min(std::min(g[DG_NROWS], h->drows_cap), (i64)capacity);
    if (rows && m > 0) CK(h, cudaMemcpy(rows, h->drows.p, (size_t)m * 7 * sizeof(i64), cudaMemcpyDeviceToHost));
    return RSIM_OK;
}

// diagnostics (RSIM_DET_DEBUG set at rsim_load_detector): per decision code, holders, min / sum
// holder-free product, chosen hit tokens, chosen product, chosen held, listed tracks
rsim_status rsim_detector_debug(rsim_t *h, int64_t *out, int64_t n) {
    if (!h || !h->ddbg.p) return RSIM_E_INVALID;
    CK(h, cudaMemcpy(out, h->ddbg.p, (size_t)std::min<i64>(n, h->R) * (8 + h->N) * sizeof(i64), cudaMemcpyDeviceToHost));
    return RSIM_OK;
}

// ---------------------------------------------------------------- generate_synthetic
// The reference's trace generator (trace.py:218-268) on the device: rsim_synth.cuh.
struct rsim_synth {
    int device = 0;
    i64 n = 0, nb = 0;
    double *arrival = nullptr;
    u64 *rid = nullptr, *ckey = nullptr, *blocks = nullptr;
    i64 *in_tok = nullptr, *out_tok = nullptr, *blk_off = nullptr;
};

static rsim_status synth_fail(rsim_status st, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_create_err, sizeof(g_create_err), fmt, ap);
    va_end(ap);
    return st;
}

void rsim_synth_free(rsim_synth_t *g) {
    if (!g) return;
    cudaSetDevice(g->device);
    for (void *p : {(void *)g->arrival, (void *)g->rid, (void *)g->ckey, (void *)g->blocks, (void *)g->in_tok,
                    (void *)g->out_tok, (void *)g->blk_off})
        if (p) cudaFreeAsync(p, 0);
    cudaStreamSynchronize(0);
    delete g;
}

rsim_status rsim_synth_generate(const rsim_synth_class *classes, int32_t n_classes, double duration_s,
                                double mean_rate_rps, uint64_t seed, int64_t block_size, int32_t device,
                                rsim_synth_t **out, int64_t *n_requests, int64_t *n_blocks) {
    if (!out || !classes) return synth_fail(RSIM_E_INVALID, "null argument");
    *out = nullptr;
    // SyntheticSpec.validate (trace.py:86-100)
    if (!(duration_s > 0) || !(mean_rate_rps > 0) || block_size < 1)
        return synth_fail(RSIM_E_TRACE, "duration, rate, and block size must be positive");
    if (n_classes < 1) return synth_fail(RSIM_E_TRACE, "at least one request class is required");
    double total = 0.0;
    for (int c = 0; c < n_classes; c++) total += classes[c].weight;
    if (std::fabs(total - 1.0) > 1e-9) return synth_fail(RSIM_E_TRACE, "class weights must sum to 1.0, got %.17g", total);
    std::vector<SynClass> hc(n_classes);
    for (int c = 0; c < n_classes; c++) {
        const rsim_synth_class &k = classes[c];
        if (!(k.weight > 0)) return synth_fail(RSIM_E_TRACE, "class weights must be positive");
        if (k.shared_blocks < 0 || k.suffix_lo < 0) return synth_fail(RSIM_E_TRACE, "block counts must be non-negative");
        if (k.shared_blocks + k.suffix_lo < 1) return synth_fail(RSIM_E_TRACE, "each request needs at least one block");
        if (k.suffix_lo > k.suffix_hi) return synth_fail(RSIM_E_TRACE, "suffix_blocks range is inverted");
        if (k.output_lo < 1 || k.output_lo > k.output_hi)
            return synth_fail(RSIM_E_TRACE, "output_tokens range must be >= 1 and ordered");
        if (k.suffix_hi - k.suffix_lo >= (1ll << 31) || k.output_hi - k.output_lo >= (1ll << 31) ||
            k.shared_blocks + k.suffix_hi >= (1ll << 31) || k.output_hi >= (1ll << 31))
            return synth_fail(RSIM_E_UNSUPPORTED, "size ranges wider than 2^31 are not generated on the device");
        hc[c] = SynClass{k.weight * mean_rate_rps, k.shared_blocks, k.suffix_lo, k.suffix_hi, k.output_lo, k.output_hi};
    }
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return synth_fail(RSIM_E_CUDA, "cudaSetDevice: %s", cudaGetErrorString(e));
    rsim_synth_t *g = new rsim_synth_t();
    g->device = device;
    SynClass *dcls = nullptr;
    i64 *dtoff = nullptr, *dcount = nullptr, *dcoff = nullptr, *row_seq = nullptr, *row_len = nullptr;
    int *nsuf = nullptr, *nout = nullptr, *row_cls = nullptr;
    double *times = nullptr;
    void *tmp = nullptr;
    cudaStream_t s = nullptr;
    rsim_status st = RSIM_OK;
    std::vector<i64> toff(n_classes + 1, 0), cnt(n_classes, 0), coff(n_classes + 1, 0);
#define SY(call)                                                                                   \
    do {                                                                                           \
        cudaError_t _e = (call);                                                                   \
        if (_e != cudaSuccess) { st = synth_fail(RSIM_E_CUDA, "%s: %s", #call, cudaGetErrorString(_e)); goto done; } \
    } while (0)
    SY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    {   // stream-ordered allocations from the device pool, kept across calls (no cudaMalloc /
        // cudaFree device syncs for the ~0.3 GB a 1M-request trace takes)
        cudaMemPool_t pool;
        uint64_t keep = ~0ull;
        SY(cudaDeviceGetDefaultMemPool(&pool, device));
        SY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    }
    SY(cudaMallocAsync(&dcls, n_classes * sizeof(SynClass), s));
    SY(cudaMemcpyAsync(dcls, hc.data(), n_classes * sizeof(SynClass), cudaMemcpyHostToDevice, s));
    SY(cudaMallocAsync(&dtoff, (n_classes + 1) * sizeof(i64), s));
    SY(cudaMallocAsync(&dcoff, (n_classes + 1) * sizeof(i64), s));
    SY(cudaMallocAsync(&dcount, n_classes * sizeof(i64), s));
    for (int c = 0; c < n_classes; c++) {      // Poisson(rate * duration) + 12 sigma; a rerun if short
        const double lam = hc[c].rate * duration_s;
        toff[c + 1] = toff[c] + (getenv("RSIM_SYNTH_TIGHT") ? 1 : (i64)std::ceil(lam + 12.0 * std::sqrt(lam) + 64.0));
    }                                          // (RSIM_SYNTH_TIGHT: tests force the rerun pass)
    for (int pass = 0; pass < 2; pass++) {
        if (times) { cudaFreeAsync(times, s); times = nullptr; }
        SY(cudaMallocAsync(&times, std::max<i64>(toff[n_classes], 1) * sizeof(double), s));
        SY(cudaMemcpyAsync(dtoff, toff.data(), (n_classes + 1) * sizeof(i64), cudaMemcpyHostToDevice, s));
        synth_arrivals_kernel<<<n_classes, 32, 0, s>>>(dcls, seed, duration_s, dtoff, times, dcount);
        SY(cudaGetLastError());
        SY(cudaMemcpyAsync(cnt.data(), dcount, n_classes * sizeof(i64), cudaMemcpyDeviceToHost, s));
        SY(cudaStreamSynchronize(s));
        bool fits = true;
        for (int c = 0; c < n_classes; c++) fits &= cnt[c] <= toff[c + 1] - toff[c];
        if (fits) break;
        for (int c = 0; c < n_classes; c++) toff[c + 1] = toff[c] + cnt[c];
    }
    for (int c = 0; c < n_classes; c++) coff[c + 1] = coff[c] + cnt[c];
    g->n = coff[n_classes];
    {
        const i64 n = g->n, n1 = std::max<i64>(n, 1);
        SY(cudaMemcpyAsync(dcoff, coff.data(), (n_classes + 1) * sizeof(i64), cudaMemcpyHostToDevice, s));
        SY(cudaMallocAsync(&nsuf, n1 * sizeof(int), s));
        SY(cudaMallocAsync(&nout, n1 * sizeof(int), s));
        SY(cudaMallocAsync(&row_cls, n1 * sizeof(int), s));
        SY(cudaMallocAsync(&row_seq, n1 * sizeof(i64), s));
        SY(cudaMallocAsync(&row_len, n1 * sizeof(i64), s));
        SY(cudaMallocAsync(&g->arrival, n1 * sizeof(double), s));
        SY(cudaMallocAsync(&g->out_tok, n1 * sizeof(i64), s));
        SY(cudaMallocAsync(&g->in_tok, n1 * sizeof(i64), s));
        SY(cudaMallocAsync(&g->rid, n1 * sizeof(u64), s));
        SY(cudaMallocAsync(&g->ckey, n1 * sizeof(u64), s));
        SY(cudaMallocAsync(&g->blk_off, (n + 1) * sizeof(i64), s));
        SY(cudaMemsetAsync(g->blk_off, 0, sizeof(i64), s));
        if (n > 0) {
            synth_sizes_kernel<<<n_classes, 32, 0, s>>>(dcls, seed, dcoff, nsuf, nout);
            SY(cudaGetLastError());
            synth_order_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(dcls, n_classes, dtoff, dcoff, times, nsuf,
                                                                          nout, n, g->arrival, row_cls, row_seq,
                                                                          row_len, g->out_tok);
            SY(cudaGetLastError());
            size_t tb = 0;
            SY(cub::DeviceScan::InclusiveSum(nullptr, tb, row_len, g->blk_off + 1, (int)n, s));
            SY(cudaMallocAsync(&tmp, tb, s));
            SY(cub::DeviceScan::InclusiveSum(tmp, tb, row_len, g->blk_off + 1, (int)n, s));
        }
        SY(cudaMemcpyAsync(&g->nb, g->blk_off + n, sizeof(i64), cudaMemcpyDeviceToHost, s));
        SY(cudaStreamSynchronize(s));
        SY(cudaMallocAsync(&g->blocks, std::max<i64>(g->nb, 1) * sizeof(u64), s));
        if (n > 0) {
            synth_blocks_kernel<<<(unsigned)((n + 7) / 8), 256, 0, s>>>(dcls, seed, n, block_size, row_cls, row_seq,
                                                                       g->blk_off, g->blocks, g->rid, g->in_tok,
                                                                       g->ckey);
            SY(cudaGetLastError());
        }
        SY(cudaStreamSynchronize(s));
    }
#undef SY
done:
    for (void *p : {(void *)dcls, (void *)dtoff, (void *)dcount, (void *)dcoff, (void *)row_seq, (void *)row_len,
                    (void *)nsuf, (void *)nout, (void *)row_cls, (void *)times, tmp})
        if (p) cudaFreeAsync(p, s);
    if (s) { cudaStreamSynchronize(s); cudaStreamDestroy(s); }
    if (st != RSIM_OK) { rsim_synth_free(g); return st; }
    *out = g;
    if (n_requests) *n_requests = g->n;
    if (n_blocks) *n_blocks = g->nb;
    return RSIM_OK;
}

rsim_status rsim_synth_read(const rsim_synth_t *g, uint64_t *request_id, double *arrival_s, int64_t *in_tokens,
                            int64_t *out_tokens, uint64_t *class_key, int64_t *blk_off, uint64_t *blocks) {
    if (!g) return synth_fail(RSIM_E_INVALID, "null generator");
    cudaError_t e = cudaSetDevice(g->device);
    const size_t n = (size_t)g->n;
    struct { void *dst; const void *src; size_t bytes; } cp[] = {
        {request_id, g->rid, n * 8}, {arrival_s, g->arrival, n * 8}, {in_tokens, g->in_tok, n * 8},
        {out_tokens, g->out_tok, n * 8}, {class_key, g->ckey, n * 8}, {blk_off, g->blk_off, (n + 1) * 8},
        {blocks, g->blocks, (size_t)g->nb * 8}};
    for (auto &c : cp)
        if (e == cudaSuccess && c.dst && c.bytes) e = cudaMemcpy(c.dst, c.src, c.bytes, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return synth_fail(RSIM_E_CUDA, "rsim_synth_read: %s", cudaGetErrorString(e));
    return RSIM_OK;
}

rsim_status rsim_synth_device_arrays(const rsim_synth_t *g, const void **arrays) {
    if (!g || !arrays) return synth_fail(RSIM_E_INVALID, "null argument");
    const void *a[7] = {g->rid, g->arrival, g->in_tok, g->out_tok, g->ckey, g->blk_off, g->blocks};
    for (int i = 0; i < 7; i++) arrays[i] = a[i];
    return RSIM_OK;
}
