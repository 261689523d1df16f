/* rsim_io.h -- trace codec of librsimio (host C++, no CUDA): the reference's JSONL trace
 * format parsed straight into the packed SoA/CSR arrays rsim_load_trace takes.
 *
 * Replaces the per-line Python parse of the reference's load_trace
 * (/root/reference/pkg/src/routesim/trace.py:108-167: _parse_line + load_trace), which
 * builds one TraceRecord object per line -- the slow path at 1M-line traces (SURVEY 8f
 * rank 4). Same acceptance rules, checks in the same order, same error texts; the
 * caller (paper_2603_15202_b200/trace.py: load_trace_packed) reads the file and raises
 * the reference's TraceError from the status below.
 *
 * Deliberate limits: an id or in/out token count that does not fit the packed 64-bit
 * columns (the reference accepts any Python int) is RSIM_IO_UNSUPPORTED. */
#ifndef RSIM_IO_H
#define RSIM_IO_H
#include <stdint.h>
#include <stddef.h>
#ifdef __cplusplus
extern "C" {
#endif

enum {
    RSIM_IO_OK = 0,
    RSIM_IO_JSON = 1,          /* json.loads failed: message = JSONDecodeError.msg        */
    RSIM_IO_RECORD = 2,        /* a field check of _parse_line failed: message = its text */
    RSIM_IO_ORDER = 3,         /* arrival before the previous one (load_trace)           */
    RSIM_IO_UNSUPPORTED = 4    /* value outside the packed columns' range                */
};

typedef struct rsim_trace_parse rsim_trace_parse;

/* Parse a whole UTF-8 JSONL buffer (the file's bytes). Lines are split and blank lines
 * skipped as str.splitlines / str.strip do. *out is always set (free it); the status is
 * also returned by rsim_trace_parse_status. */
int rsim_trace_parse_jsonl(const char *buf, int64_t len, rsim_trace_parse **out);
int rsim_trace_parse_status(const rsim_trace_parse *p);
/* Records and total prefix blocks parsed. */
int64_t rsim_trace_parse_count(const rsim_trace_parse *p, int64_t *n_blocks);
/* Copy the columns out (caller-allocated: R entries, blk_off R+1, blocks n_blocks). class_key
 * is the record's "class" or, when absent / null, class_key(blocks) (detector.py:41-45). */
void rsim_trace_parse_copy(const rsim_trace_parse *p, uint64_t *request_id, double *arrival_s,
                           int64_t *in_tokens, int64_t *out_tokens, uint64_t *class_key,
                           int64_t *blk_off, uint64_t *blocks);
/* On failure: the message, the 1-based line, and for RSIM_IO_ORDER the two arrivals. */
const char *rsim_trace_parse_error(const rsim_trace_parse *p, int64_t *line, double *arrival, double *previous);
void rsim_trace_parse_free(rsim_trace_parse *p);

#ifdef __cplusplus
}
#endif
#endif
