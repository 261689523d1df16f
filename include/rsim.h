/*
 * rsim.h -- C ABI of librsim, the B200-native multiplicative router.
 *
 * The reference (routesim, pure Python) has no FFI; each entry point below
 * replaces one Python call on the routing hot path and is what a ctypes /
 * cffi binding of the reference's ClusterSim would bind.
 *
 * Conventions: every call returns an rsim_status (0 = ok). Inputs are plain
 * host pointers copied on entry; outputs are caller-allocated host buffers
 * filled before return; no pointer is retained. A handle owns one CUDA
 * device context + stream and is not thread-safe. There is no CPU fallback:
 * without a usable sm_100 device rsim_create fails with RSIM_E_CUDA.
 */
#ifndef RSIM_H
#define RSIM_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    RSIM_OK = 0,
    RSIM_E_INVALID = 1,        /* bad argument / config (reference: ValueError, cluster.py:36-64) */
    RSIM_E_TRACE = 2,          /* malformed trace (reference: TraceError, trace.py:30-38)          */
    RSIM_E_CACHE_FULL = 3,     /* pinned blocks exceed capacity (reference: CacheFullError, kvcache.py:163) */
    RSIM_E_DUPLICATE = 4,      /* request enqueued twice (reference: DuplicateRequestError, engine.py:266) */
    RSIM_E_INVARIANT = 5,      /* device consistency check failed (reference: InvariantError / unpin ValueError) */
    RSIM_E_CUDA = 6,           /* CUDA runtime / launch failure                                    */
    RSIM_E_QUEUE_OVERFLOW = 7, /* per-instance queue ring full: recreate with larger queue_capacity */
    RSIM_E_TABLE_FULL = 8,     /* per-instance KV$ hash table too small: recreate with larger table */
    RSIM_E_UNSUPPORTED = 9,    /* feature outside the device path (detector, staleness > 0, ...)  */
    RSIM_E_COMM = 10,          /* multi-GPU exchange failure                                        */
    RSIM_E_NO_INSTANCES = 11,  /* empty candidate set (reference: NoInstancesError, policies.py:226) */
    RSIM_E_HISTORY_OVERFLOW = 12, /* view-history ring full (staleness > 0): recreate with larger history_capacity */
    RSIM_E_DETECTOR = 13       /* detector capacity exceeded (classes re-evaluated in one decision > 64)  */
} rsim_status;

enum { RSIM_POLICY_MULTIPLICATIVE = 0, RSIM_POLICY_VLLM = 1, RSIM_POLICY_LEAST_BS = 2,
       RSIM_POLICY_LINEAR = 3, RSIM_POLICY_FILTER = 4,
       RSIM_POLICY_SIMULATE = 5 };   /* policies.py:104-192; simulate: estimate_ttft_us, policies.py:142-157 */
enum { RSIM_KV_P_TOKENS = 0, RSIM_KV_ONE_MINUS_HIT = 1 };
enum { RSIM_BAL_BS = 0, RSIM_BAL_TOTAL_TOKENS = 1 };

/* Mirrors ClusterConfig + CostModel + CacheConfig + PolicyConfig
 * (reference cluster.py:32-64, engine.py:46-55, policies.py:37-53). */
#define RSIM_ABI_VERSION 2
typedef struct rsim_config {
    uint32_t struct_size;           /* = sizeof(rsim_config) as the caller compiled it: rsim_create
                                       rejects a mismatch (a binding built against another layout) */
    uint32_t abi_version;           /* = RSIM_ABI_VERSION                                       */
    int32_t n_instances;            /* ClusterConfig.n_instances                              */
    int32_t block_size;             /* CacheConfig.block_size                                 */
    int64_t capacity_blocks;        /* CacheConfig.capacity_blocks, -1 = infinite (None)      */
    double prefill_base_ms, prefill_per_token_ms;             /* CostModel                    */
    double decode_base_ms, decode_per_seq_ms, decode_per_ctx_token_ms;
    int64_t chunk_tokens, max_batch_requests;
    int32_t policy;                 /* RSIM_POLICY_*                                           */
    int32_t kv_indicator;           /* RSIM_KV_*   (multiplicative)                            */
    int32_t balance_indicator;      /* RSIM_BAL_*  (multiplicative)                            */
    int32_t debug_checks;           /* ClusterConfig.debug_checks: replay one decision per launch and
                                       check InstanceSim.reconcile + PrefixCache.check_invariants on
                                       device after each (cluster.py:168-170) -> RSIM_E_INVARIANT   */
    double q_weight;                /* PolicyConfig.q_weight (vllm)                            */
    uint64_t tie_seed_lo, tie_seed_hi; /* TieBreaker counter = stable_key(seed, tie_break_seed), cluster.py:90-94 */
    int32_t device;                 /* CUDA ordinal                                            */
    int32_t queue_capacity;         /* per-instance queue ring entries, 0 = auto               */
    int32_t table_slots_log2;       /* per-instance KV$ table slots (log2), 0 = auto           */
    int32_t ctas;                   /* replay cluster size (1..16), 0 = auto                   */
    int32_t warps_per_cta;          /* 0 = auto                                                */
    int32_t record_steps;           /* keep the per-step log (RunReport.steps / bs_series)     */
    int64_t step_log_capacity;      /* records, 0 = auto                                       */
    int64_t expected_keys;          /* sizing hint: upper bound on keys one instance holds, 0 = from trace */
    /* Multi-GPU sharding: n_instances is the GLOBAL cluster size; this handle owns
     * the contiguous shard [lo, hi) of rank `rank` of `world` (sizes differ by at most one).
     * Every decision exchanges one (min score, tie count) partial per rank through peer-mapped
     * mailboxes (rsim_set_peer / rsim_open_peer_ipc); all ranks replay collectively. */
    int32_t world;                  /* ranks sharing the cluster (1 = unsharded), <= 8         */
    int32_t rank;
    int64_t comm_timeout_ms;        /* a rank waiting longer on a peer fails with RSIM_E_COMM  */
    int64_t runs_capacity;          /* per-instance touch-run ring (finite capacity), 0 = auto */
    double kv_weight;               /* PolicyConfig.kv_weight (linear)                         */
    double bs_norm_cap;             /* PolicyConfig.bs_norm_cap (linear); 0 = per-decision max */
    int64_t range_threshold;        /* PolicyConfig.range_threshold (filter)                   */
    int64_t staleness_us;           /* ClusterSim.staleness_us = round(staleness_ms * 1000), cluster.py:77;
                                       scores see each instance's view as of now - staleness      */
    int32_t history_capacity;       /* per-instance view-history ring entries (staleness > 0), 0 = auto */
    int32_t reserved0;
    /* Prefix-hotspot detector (DetectorConfig, detector.py:104-119; ClusterConfig.detector). Trace
     * replays run it on one GPU with multiplicative / vllm / least_bs / capped linear scores;
     * classes come from rsim_load_detector. det_on = 0: no detector (None). */
    int32_t det_on;
    int32_t det_top_k_classes;
    int32_t det_class_key_blocks;
    int32_t det_mitigation;         /* 0 exclude_holders, 1 force_least_bs                    */
    int32_t det_compare_mean_non_holder;
    int32_t reserved1;
    double det_window_s;
    double det_consecutive_multiplier;
    /* simulate policy: Policy.sim_cost_model (policies.py:206-211) -- the CostModel coefficients the
     * TTFT replay uses (CostModel.scaled(mis_tuned_factor) when mis-tuned, else the engine's own) */
    double sim_prefill_base_ms, sim_prefill_per_token_ms;
    double sim_decode_base_ms, sim_decode_per_seq_ms, sim_decode_per_ctx_token_ms;
} rsim_config;

typedef struct rsim rsim_t;

/* sizeof(rsim_config) of this build: bindings assert it before the first rsim_create. */
size_t rsim_config_size(void);

/* ClusterSim.__init__ (cluster.py:73-102): allocate device state for N instances. */
rsim_status rsim_create(const rsim_config *cfg, rsim_t **out);
void rsim_destroy(rsim_t *h);
/* Last error message of the handle (or of the last failed create when h == NULL). */
const char *rsim_last_error(const rsim_t *h);
/* Clear all instance, KV$ and tie-break state back to ClusterSim.__init__'s. */
rsim_status rsim_reset(rsim_t *h);

/* run_trace's input (cluster.py:172-201 + TraceRecord, trace.py:42-54), CSR-packed:
 * request i has blocks[blk_off[i] .. blk_off[i+1]). arrival_us = round(arrival_s*1e6).
 * Copies to HBM and runs the chain-hash kernel (hashing.chain_keys, hashing.py:36-47,
 * plus the output-block keys of engine.py:363-372) over every request. */
rsim_status rsim_load_trace(rsim_t *h, int64_t n_requests, const int64_t *arrival_us,
                            const int64_t *input_tokens, const int64_t *output_tokens,
                            const uint64_t *request_id, const int64_t *blk_off,
                            const uint64_t *blocks);

/* _loop_parallel's body (cluster.py:244-287) for decisions [first, first+count):
 * per arrival, advance every instance through steps starting before it, then
 * route (cluster.py:130-154) and enqueue on the winner -- entirely on device. */
rsim_status rsim_replay(rsim_t *h, int64_t first, int64_t count);
/* drain(until) (cluster.py:250-273); until = INT64_MAX runs every instance to idle. */
rsim_status rsim_drain(rsim_t *h, int64_t until_us);

/* Outputs of the loaded trace (RequestMetrics, metrics.py:31-41); -1 = not reached. */
rsim_status rsim_read_decisions(rsim_t *h, int64_t first, int64_t count,
                                int32_t *chosen_instance, int64_t *hit_tokens);
rsim_status rsim_read_request_times(rsim_t *h, int64_t first, int64_t count,
                                    int64_t *first_sched_us, int64_t *first_token_us,
                                    int64_t *finish_us);
/* Per-instance state: 12 int64 per instance:
 * r_bs, q_bs, pending, total, dc (live), view r, q, pending, total, dc, busy_until_us, occupancy. */
rsim_status rsim_read_instances(rsim_t *h, int64_t *out12xN);
/* Step log: 6 int64 per record (instance, start_us, end_us, prefill_us, bs_after, step_index),
 * unordered. With out = NULL, *n_records receives an upper bound of the record count (records
 * are reserved per device warp in chunks; a bound above cap: RSIM_E_INVALID); with out, the
 * records written (the unused reserved ones dropped). */
rsim_status rsim_read_step_log(rsim_t *h, int64_t *out, int64_t cap, int64_t *n_records);
/* Per-request batch size right after its enqueue (Collector.record_bs at route, cluster.py:152). */
rsim_status rsim_read_route_bs(rsim_t *h, int64_t first, int64_t count, int64_t *bs);

/* One ClusterSim.route(record, now_us) call WITHOUT advancing engine steps
 * (cluster.py:130-154) on loaded request r. scores (N doubles) may be NULL. */
rsim_status rsim_route_one(rsim_t *h, int64_t r, int64_t now_us, int32_t *chosen,
                           int64_t *hit_tokens, double *scores);
/* route() of a request id already present on some instances (InstanceSim._present, engine.py:266-267):
 * the decision is made as usual (the TieBreaker counter moves); if the winner is one of
 * holders[0..n_holders) (global ids) nothing is enqueued and RSIM_E_DUPLICATE is returned. */
rsim_status rsim_route_one_excl(rsim_t *h, int64_t r, int64_t now_us, const int32_t *holders, int32_t n_holders,
                                int32_t *chosen, int64_t *hit_tokens, double *scores);
/* ClusterSim.route(record, now_us) of a request that is not loaded yet (cluster.py:130-154):
 * scores (N, may be NULL) are RoutingDecision.scores, NaN for a candidate the detector excluded;
 * branch (may be NULL) receives the detector verdict applied (0 none, 2 holders excluded, 3 forced
 * least_bs, 4 excluded + route_filter's batch-size branch). One launch (route_kernel) for the plain
 * policies on <= 256 instances, else three. Otherwise as follows:
 * appends it to the loaded trace (as rsim_load_trace of one request would) and decides it, with
 * the holders semantics of rsim_route_one_excl -- one fused call (the request goes in and the
 * decision comes out through mapped pinned memory, three launches, one stream synchronisation). */
rsim_status rsim_route_request(rsim_t *h, int64_t now_us, int64_t input_tokens, int64_t output_tokens,
                               uint64_t request_id, const uint64_t *blocks, int64_t n_blocks,
                               const int32_t *holders, int32_t n_holders, int32_t *chosen, int64_t *hit_tokens,
                               double *scores, int32_t *branch);
/* route() with the hotspot detector (cluster.py:133-139: verdict before choose, observe after the
 * enqueue): the class of the request the next rsim_route_request appends -- its track, numbered
 * densely by first arrival (track == the current track count opens a new one, whose exemplar is
 * that request's first exemplar_len chain keys; detector.py:303-307) and class key -- and the
 * DetectorRows to keep room for (window rolls so far + 1, times top_k). */
rsim_status rsim_detector_next(rsim_t *h, int32_t track, int32_t exemplar_len, uint64_t class_key,
                               int64_t rows_capacity);
/* InstanceSim.queue / .running (engine.py:212-213) of a local instance: 8 int64 per slot -- the FIFO
 * queue in order, then the running list: request index, kind (0 queued / 1 running), pending,
 * generated, hit blocks, input tokens, output tokens, flags (bit0: prefill scheduled). out may be
 * NULL to query the counts. */
rsim_status rsim_read_slots(rsim_t *h, int32_t instance, int64_t *out, int64_t cap, int64_t *n_queued,
                            int64_t *n_running);
/* Start of a run_trace on a handle with API state: no instance has a step scheduled
 * (cluster.py:210-211, 247); queued requests wait for an arrival routed to their instance. */
rsim_status rsim_unschedule(rsim_t *h);
/* InstanceSim.enqueue(record r, now_us) on a given instance (engine.py:262-289). */
rsim_status rsim_enqueue(rsim_t *h, int32_t instance, int64_t r, int64_t now_us, int64_t *hit_tokens);

/* PrefixCache on one instance (kvcache.py:65-104), keys = chain keys. */
rsim_status rsim_cache_insert_keys(rsim_t *h, int32_t instance, const uint64_t *keys, int64_t n,
                                   int64_t now_us, int64_t *evicted);
rsim_status rsim_cache_match_keys(rsim_t *h, int32_t instance, const uint64_t *keys, int64_t n,
                                  int64_t *hit_blocks);

/* Batched what-if probe (no commits): hit blocks of requests [first, first+count) on
 * every instance against the current state -> out[count x N] (int32). */
rsim_status rsim_probe_batch(rsim_t *h, int64_t first, int64_t count, int32_t *hit_blocks_out);

/* hashing.chain_keys on the device (K1) for an ad-hoc block list. */
rsim_status rsim_chain_keys(rsim_t *h, const uint64_t *blocks, int64_t n, uint64_t *keys_out);

/* Timing of the last rsim_replay / rsim_drain / K1 launch (CUDA events on the handle's stream). */
rsim_status rsim_last_timings(rsim_t *h, double *replay_ms, double *k1_ms, double *drain_ms);
/* Per-decision device timestamps (%globaltimer ns) of the last replay, count entries. */
rsim_status rsim_read_decision_ns(rsim_t *h, int64_t first, int64_t count, int64_t *ns);
/* Resident re-run (bench "value"): reset engine/KV$/tie state, rerun K1 over the
 * loaded trace, replay every decision and drain to idle; *device_ms = CUDA-event
 * time of the whole sequence on the handle's stream. Equals reset+K1+replay+drain. */
rsim_status rsim_rerun(rsim_t *h, double *device_ms);
/* Counters of the last replay (16 int64): [0] algorithmic probe bytes (8*B per
 * decision + sum_i 8*min(h_i+1,B) + 16 per instance probed), [1] engine steps, [2] SM cycles
 * in engine steps, [3] SM cycles finishing requests, [4] requests loaded, [5] blocks,
 * [6] finisher batches, [7] local instances,
 * [8..15] SM cycles of CTA 0 / warp 0 per decision phase: staging wait, drain, probe,
 * publish + speculative drain, exchange wait, decide, barrier, commit. */
rsim_status rsim_read_counters(rsim_t *h, int64_t *out16);
/* Sharded replay plumbing. The mailbox is device memory peers write into. */
rsim_status rsim_shard_bounds(const rsim_t *h, int32_t *lo, int32_t *hi);
rsim_status rsim_mailbox(rsim_t *h, void **dev_ptr);
rsim_status rsim_mailbox_ipc_handle(rsim_t *h, unsigned char out64[64]);   /* cudaIpcGetMemHandle */
rsim_status rsim_set_peer(rsim_t *h, int32_t rank, void *peer_mailbox);    /* same-process peer    */
rsim_status rsim_open_peer_ipc(rsim_t *h, int32_t rank, const unsigned char in64[64]);
/* Diagnostics: record, for the first capacity_decisions decisions of each replay launch, one
 * 8 x uint16 record per (decision, instance warp): [0] cycles/16 from the warp's release to its
 * partial, [1] drain cycles/16, [2] probe+score cycles/16, [3] staging wait cycles/16, [4] engine
 * steps, [5] finisher batches, [6] instances served by the probe-ahead, [7] instances of the warp.
 * capacity 0 turns recording off. Read back with rsim_read_phase_records. */
rsim_status rsim_phase_records(rsim_t *h, int64_t capacity_decisions);
rsim_status rsim_read_phase_records(rsim_t *h, uint16_t *out, int64_t n_decisions, int32_t *warps_per_decision);
/* Diagnostics (-DRSIM_DIAG builds): per decision, %globaltimer of every instance warp's publish
 * ([C*W]), then CTA 0's control warp: partials landed, decided; CTA 0 warp 0: released; 0. */
rsim_status rsim_read_phase_times(rsim_t *h, uint64_t *out, int64_t n_decisions);
/* Diagnostics of builds with -DRSIM_DIAG -DRSIM_STEP_PROFILE (32 int64): [0..7] SM cycles summed
 * over engine steps per step section (setup, plan, cost, apply, pops, decode, finishers,
 * joins+tail); [8..9] count / cycles of steps where a request finishes, [10..11] of other full
 * steps, [12..13] of pure decode steps; [14..15] warp 0 of CTA 0: advancing non-candidates /
 * probe-ahead cycles; [16..19] its probe-ahead sections (setup, issue, evaluate, tail); zeros
 * otherwise. */
rsim_status rsim_read_step_cycles(rsim_t *h, int64_t *out32);
/* ClusterConfig.debug_checks' per-step checks, run now over every instance of the handle
 * (engine.py:248-258 reconcile, kvcache.py:178-194 check_invariants); RSIM_E_INVARIANT with the
 * instance and the failed check in rsim_last_error. Runs automatically after every decision and
 * after the drain when cfg.debug_checks is set. */
rsim_status rsim_check_invariants(rsim_t *h);
/* Fault injection for the checker's tests: what = 0 pins the deepest KV$ entry of the local
 * instance once more (its parent no longer covers the pin), 1 breaks the live aggregates,
 * 2 ages the deepest entry's parent. */
rsim_status rsim_debug_corrupt(rsim_t *h, int32_t instance, int32_t what);
/* Number of kernels librsim launched since create (evidence for bench gpu_launches). */
int64_t rsim_launch_count(const rsim_t *h);

/* ---- prefix-hotspot detector (reference detector.py; cluster.py:131-140, 194-201) ---- */
/* Classes of the loaded trace (all n requests, loaded by one rsim_load_trace after a reset):
 * track_of_request[r] = dense class id numbered by first arrival; per class the exemplar
 * (its first request's leading min(class_key_blocks, B) chain keys: offset into the loaded
 * blocks, length) and its class_key (detector.py:41-45). rows_capacity bounds the DetectorRows
 * kept (windows x top_k_classes + top_k_classes is always enough). */
rsim_status rsim_load_detector(rsim_t *h, int64_t n, const int32_t *track_of_request, int32_t n_tracks,
                               const int64_t *exemplar_offset, const int32_t *exemplar_len,
                               const uint64_t *class_key, int64_t rows_capacity);
/* Detector.finalize (detector.py:373-377): the last window's rows, on the tables after the drain. */
rsim_status rsim_detector_finalize(rsim_t *h);
/* DetectorRows, 7 int64 each: window_start_s (f64 bits), class_key, fraction (f64 bits),
 * n_holders, n_others, suspect, phase; first_violation_us = -1 for None. */
rsim_status rsim_read_detector(rsim_t *h, int64_t *rows, int64_t capacity, int64_t *n_rows,
                               int64_t *first_violation_us);
/* Diagnostics: 8 words per decision when RSIM_DET_DEBUG was set at rsim_load_detector. */
rsim_status rsim_detector_debug(rsim_t *h, int64_t *out, int64_t n);

/* ---- synthetic traces on the device (reference trace.py:218-268 generate_synthetic) ---- */
/* One ClassSpec (trace.py:58-69): weight, shared_blocks, suffix_blocks = [suffix_lo, suffix_hi],
 * output_tokens = [output_lo, output_hi] (inclusive ranges, each narrower than 2^31). */
typedef struct {
    double weight;
    int64_t shared_blocks;
    int64_t suffix_lo, suffix_hi;
    int64_t output_lo, output_hi;
} rsim_synth_class;
typedef struct rsim_synth rsim_synth_t;
/* generate_synthetic(SyntheticSpec(duration_s, mean_rate_rps, classes, seed, block_size)) on
 * `device`, bit-identical to the reference's records (the same random.Random streams, draw
 * order, (t, class, seq) sort and stable_key hashes; glibc's log for expovariate). Spec errors
 * are the reference's TraceError messages (RSIM_E_TRACE). The trace stays in device memory
 * until rsim_synth_free; *n_requests / *n_blocks size the rsim_synth_read buffers. Messages
 * go to rsim_last_error(NULL). seed = the spec's seed mod 2^64. Replaces the reference's
 * generate_synthetic (trace.py:218), which the Python mirror calls
 * paper_2603_15202_b200.trace.generate_synthetic_device. */
rsim_status rsim_synth_generate(const rsim_synth_class *classes, int32_t n_classes, double duration_s,
                                double mean_rate_rps, uint64_t seed, int64_t block_size, int32_t device,
                                rsim_synth_t **out, int64_t *n_requests, int64_t *n_blocks);
/* Host copies of the PackedTrace columns (any pointer may be NULL): request_id[n], arrival_s[n],
 * in_tokens[n], out_tokens[n], class_key[n], blk_off[n+1], blocks[n_blocks]. */
rsim_status rsim_synth_read(const rsim_synth_t *g, uint64_t *request_id, double *arrival_s, int64_t *in_tokens,
                            int64_t *out_tokens, uint64_t *class_key, int64_t *blk_off, uint64_t *blocks);
/* The same seven columns' device pointers (valid until rsim_synth_free). */
rsim_status rsim_synth_device_arrays(const rsim_synth_t *g, const void **arrays);
void rsim_synth_free(rsim_synth_t *g);

#ifdef __cplusplus
}
#endif
#endif /* RSIM_H */
