// rsim_io.cpp -- librsimio: the reference's JSONL trace format (trace.py:108-167) parsed in
// one pass into packed SoA/CSR columns (include/rsim_io.h). Host C++ only.
//
// Semantics followed line by line:
//   load_trace        trace.py:151-167  splitlines, skip blank (str.strip) lines, arrival order
//   _parse_line       trace.py:111-148  json.loads -> dict -> required fields -> checks in order
//   json.loads        CPython 3.12 json (scanner + decoder messages, NaN/Infinity literals,
//                     last duplicate key wins, bool is an int subclass)
//   class_key         detector.py:41-45 stable_key(0xC1A55000, *blocks[:2])
#include "../../include/rsim_io.h"

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

namespace {

inline uint64_t splitmix64(uint64_t z) {      // hashing.py:15-20
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
inline uint64_t class_key2(const uint64_t *b, size_t n) {   // stable_key(_CLASS_SALT, *b[:2])
    uint64_t acc = 0x9E3779B97F4A7C15ULL;
    acc = splitmix64(acc ^ 0xC1A55000ULL);
    for (size_t i = 0; i < n && i < 2; i++) acc = splitmix64(acc ^ b[i]);
    return acc;
}

// A JSON value as far as _parse_line looks at it.
enum Kind { K_NONE, K_NULL, K_BOOL, K_INT, K_NEGINT, K_BIGINT, K_FLOAT, K_STR, K_ARR, K_OBJ };
struct Val {
    Kind k = K_NONE;
    uint64_t u = 0;      // K_INT / K_BOOL value (non-negative, fits u64)
    double d = 0;        // float(value) of literals (NaN, +-Infinity, bools)
    const char *nb = nullptr, *ne = nullptr;   // a number's text: float() of it on demand
    double num() const {
        if (!nb) return d;
        if (k == K_INT && u < (1ULL << 53)) return (double)u;                  // exact
        char tmp[64];
        std::string big;
        const size_t n = (size_t)(ne - nb);
        const char *z;
        if (n < sizeof(tmp)) { memcpy(tmp, nb, n); tmp[n] = 0; z = tmp; } else { big.assign(nb, ne); z = big.c_str(); }
        const double x = strtod(z, nullptr);   // correctly rounded, as float(int) / float(str)
        return (k == K_INT && x == 0.0) ? 0.0 : x;                             // "-0" is the int 0
    }
};

struct Parser {
    const char *s, *e;
    const char *p;
    std::string msg;                    // JSONDecodeError.msg
    // the record's fields (last duplicate wins)
    Val id, arr, in, out, cls;
    bool has_blocks = false;
    Val blocks;                         // kind only
    std::vector<uint64_t> bv;           // block values
    bool blocks_ok = true;              // every element an int in [0, 2^64)

    void reset(const char *b, const char *end) {
        s = p = b; e = end; msg.clear();
        id = arr = in = out = cls = blocks = Val();
        has_blocks = false; bv.clear(); blocks_ok = true;
    }
    bool fail(const char *m) { if (msg.empty()) msg = m; return false; }
    void ws() { while (p < e && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) p++; }

    // JSON string (scanstring, strict): returns the decoded UTF-8 bytes when want != nullptr
    bool str(std::string *want) {
        p++;                                              // opening quote
        while (true) {
            if (p >= e) return fail("Unterminated string starting at");
            unsigned char c = (unsigned char)*p;
            if (c == '"') { p++; return true; }
            if (c < 0x20) return fail("Invalid control character at");
            if (c != '\\') { if (want) want->push_back((char)c); p++; continue; }
            p++;
            if (p >= e) return fail("Unterminated string starting at");
            char x = *p++;
            switch (x) {
                case '"': case '\\': case '/': if (want) want->push_back(x); break;
                case 'b': if (want) want->push_back('\b'); break;
                case 'f': if (want) want->push_back('\f'); break;
                case 'n': if (want) want->push_back('\n'); break;
                case 'r': if (want) want->push_back('\r'); break;
                case 't': if (want) want->push_back('\t'); break;
                case 'u': {
                    auto hex4 = [&](unsigned &v) -> bool {
                        if (e - p < 4) return false;
                        v = 0;
                        for (int i = 0; i < 4; i++) {
                            char h = p[i];
                            v <<= 4;
                            if (h >= '0' && h <= '9') v |= (unsigned)(h - '0');
                            else if (h >= 'a' && h <= 'f') v |= (unsigned)(h - 'a' + 10);
                            else if (h >= 'A' && h <= 'F') v |= (unsigned)(h - 'A' + 10);
                            else return false;
                        }
                        p += 4;
                        return true;
                    };
                    unsigned v;
                    if (!hex4(v)) return fail("Invalid \\uXXXX escape");
                    if (v >= 0xD800 && v <= 0xDBFF && e - p >= 6 && p[0] == '\\' && p[1] == 'u') {
                        const char *save = p;
                        p += 2;
                        unsigned w;
                        if (!hex4(w)) return fail("Invalid \\uXXXX escape");
                        if (w >= 0xDC00 && w <= 0xDFFF) v = 0x10000 + ((v - 0xD800) << 10) + (w - 0xDC00);
                        else p = save;
                    }
                    if (want) {                           // UTF-8 (lone surrogates as 3 bytes)
                        if (v < 0x80) want->push_back((char)v);
                        else if (v < 0x800) { want->push_back((char)(0xC0 | (v >> 6))); want->push_back((char)(0x80 | (v & 63))); }
                        else if (v < 0x10000) { want->push_back((char)(0xE0 | (v >> 12))); want->push_back((char)(0x80 | ((v >> 6) & 63))); want->push_back((char)(0x80 | (v & 63))); }
                        else { want->push_back((char)(0xF0 | (v >> 18))); want->push_back((char)(0x80 | ((v >> 12) & 63)));
                               want->push_back((char)(0x80 | ((v >> 6) & 63))); want->push_back((char)(0x80 | (v & 63))); }
                    }
                    break;
                }
                default: return fail("Invalid \\escape");
            }
        }
    }

    // number per json.scanner NUMBER_RE: (-?(?:0|[1-9]\d*))(\.\d+)?([eE][-+]?\d+)?
    bool number(Val &v) {
        const char *b = p, *q = p;
        bool neg = false;
        if (q < e && *q == '-') { neg = true; q++; }
        if (q >= e || !(*q >= '0' && *q <= '9')) return fail("Expecting value");
        if (*q == '0') q++;
        else while (q < e && *q >= '0' && *q <= '9') q++;
        const char *ie = q;
        bool isf = false;
        if (q + 1 < e && *q == '.' && q[1] >= '0' && q[1] <= '9') {
            isf = true; q += 2;
            while (q < e && *q >= '0' && *q <= '9') q++;
        }
        if (q < e && (*q == 'e' || *q == 'E')) {
            const char *r = q + 1;
            if (r < e && (*r == '+' || *r == '-')) r++;
            if (r < e && *r >= '0' && *r <= '9') {
                while (r < e && *r >= '0' && *r <= '9') r++;
                isf = true; q = r;
            }
        }
        v.nb = b; v.ne = q;
        if (isf) v.k = K_FLOAT;
        else {
            const char *dg = neg ? b + 1 : b;
            const bool zero = (ie - dg == 1 && *dg == '0');
            if (neg && !zero) v.k = K_NEGINT;
            else {
                uint64_t u = 0;
                bool big = false;
                for (const char *c = dg; c < ie; c++) {
                    const uint64_t dgt = (uint64_t)(*c - '0');
                    if (u > 1844674407370955161ULL || (u == 1844674407370955161ULL && dgt > 5)) { big = true; break; }
                    u = u * 10 + dgt;
                }
                v.k = big ? K_BIGINT : K_INT;
                v.u = big ? 0 : u;
            }
        }
        p = q;
        return true;
    }

    bool lit(const char *w) {
        const size_t n = strlen(w);
        if ((size_t)(e - p) >= n && memcmp(p, w, n) == 0) { p += n; return true; }
        return false;
    }

    // value; `field` selects where a top-level record field goes (depth 1 only)
    bool value(Val &v, int depth, bool want_elems) {
        if (p >= e) return fail("Expecting value");
        const char c = *p;
        if (c == '"') { v.k = K_STR; return str(nullptr); }
        if (c == '{') { v.k = K_OBJ; return object(depth + 1); }
        if (c == '[') { v.k = K_ARR; return array(depth + 1, want_elems); }
        if (c == 'n' && lit("null")) { v.k = K_NULL; return true; }
        if (c == 't' && lit("true")) { v.k = K_BOOL; v.u = 1; v.d = 1.0; return true; }
        if (c == 'f' && lit("false")) { v.k = K_BOOL; v.u = 0; v.d = 0.0; return true; }
        if (c == 'N' && lit("NaN")) { v.k = K_FLOAT; v.d = NAN; return true; }
        if (c == 'I' && lit("Infinity")) { v.k = K_FLOAT; v.d = INFINITY; return true; }
        if (c == '-' && lit("-Infinity")) { v.k = K_FLOAT; v.d = -INFINITY; return true; }
        if (c == '-' || (c >= '0' && c <= '9')) return number(v);
        return fail("Expecting value");
    }

    bool array(int depth, bool want_elems) {
        p++;
        ws();
        if (p < e && *p == ']') { p++; return true; }
        while (true) {
            ws();
            Val x;
            if (!value(x, depth, false)) return false;
            if (want_elems) {
                if (x.k == K_INT || x.k == K_BOOL) bv.push_back(x.u);
                else { blocks_ok = false; bv.push_back(0); }
            }
            ws();
            if (p < e && *p == ']') { p++; return true; }
            if (p < e && *p == ',') { p++; continue; }
            return fail("Expecting ',' delimiter");
        }
    }

    bool object(int depth) {
        p++;
        ws();
        if (p < e && *p == '}') { p++; return true; }
        while (true) {
            if (p >= e || *p != '"') return fail("Expecting property name enclosed in double quotes");
            std::string key;
            if (!str(depth == 1 ? &key : nullptr)) return false;
            ws();
            if (p >= e || *p != ':') return fail("Expecting ':' delimiter");
            p++;
            ws();
            Val x;
            const bool is_blocks = depth == 1 && key == "blocks";
            if (is_blocks) { bv.clear(); blocks_ok = true; }
            if (!value(x, depth, is_blocks)) return false;
            if (depth == 1) {
                if (key == "id") id = x;
                else if (key == "arrival_s") arr = x;
                else if (key == "in") in = x;
                else if (key == "out") out = x;
                else if (key == "class") cls = x;
                else if (is_blocks) { has_blocks = true; blocks = x; if (x.k != K_ARR) bv.clear(); }
            }
            ws();
            if (p < e && *p == '}') { p++; return true; }
            if (p < e && *p == ',') { p++; ws(); continue; }
            return fail("Expecting ',' delimiter");
        }
    }
};

// UTF-8 sequence at q that str.splitlines treats as a line boundary (besides \n, \r)
inline int line_break_len(const unsigned char *q, const unsigned char *e) {
    const unsigned char c = q[0];
    if (c == 0x0B || c == 0x0C || c == 0x1C || c == 0x1D || c == 0x1E) return 1;
    if (c == 0xC2 && q + 1 < e && q[1] == 0x85) return 2;
    if (c == 0xE2 && q + 2 < e && q[1] == 0x80 && (q[2] == 0xA8 || q[2] == 0xA9)) return 3;
    return 0;
}
// length of the str.isspace() character at q (0 if none); q < e
inline int space_len(const unsigned char *q, const unsigned char *e) {
    const unsigned char c = q[0];
    if (c == ' ' || (c >= 0x09 && c <= 0x0D) || (c >= 0x1C && c <= 0x1F)) return 1;
    if (c == 0xC2 && q + 1 < e && (q[1] == 0x85 || q[1] == 0xA0)) return 2;
    if (q + 2 < e) {
        if (c == 0xE1 && q[1] == 0x9A && q[2] == 0x80) return 3;
        if (c == 0xE2 && q[1] == 0x80 && ((q[2] >= 0x80 && q[2] <= 0x8A) || q[2] == 0xA8 || q[2] == 0xA9 || q[2] == 0xAF)) return 3;
        if (c == 0xE2 && q[1] == 0x81 && q[2] == 0x9F) return 3;
        if (c == 0xE3 && q[1] == 0x80 && q[2] == 0x80) return 3;
    }
    return 0;
}

struct SpecialTable {
    bool t[256];
    SpecialTable() {
        for (int i = 0; i < 256; i++) t[i] = false;
        for (int c : {0x0A, 0x0B, 0x0C, 0x0D, 0x1C, 0x1D, 0x1E, 0xC2, 0xE2}) t[c] = true;
    }
    bool operator[](unsigned char c) const { return t[c]; }
};
const SpecialTable kSpecial;

}  // namespace

struct rsim_trace_parse {
    int status = RSIM_IO_OK;
    std::string msg;
    int64_t line = 0;
    double arrival = 0, previous = 0;
    std::vector<uint64_t> id, cls, blocks;
    std::vector<double> arr;
    std::vector<int64_t> in, out, off{0};
};

extern "C" {

int rsim_trace_parse_jsonl(const char *buf, int64_t len, rsim_trace_parse **outp) {
    rsim_trace_parse *R = new rsim_trace_parse();
    *outp = R;
    const unsigned char *s = (const unsigned char *)buf, *end = s + (len > 0 ? len : 0);
    double prev = -INFINITY;
    int64_t line_no = 0;
    const unsigned char *q = s;
    Parser P;                                             // reused: its block buffer keeps its capacity
    R->blocks.reserve((size_t)(len / 24));
    auto err = [&](int st, const std::string &m) { R->status = st; R->msg = m; R->line = line_no; return st; };
    while (q < end) {
        // one line per str.splitlines
        const unsigned char *b = q, *le = q;
        int brk = 0;
        while (le < end) {
            if (!kSpecial[*le]) { le++; continue; }        // bytes that cannot start a line boundary
            if (*le == '\n' || *le == '\r') { brk = (*le == '\r' && le + 1 < end && le[1] == '\n') ? 2 : 1; break; }
            if ((brk = line_break_len(le, end)) != 0) break;
            le++;
        }
        q = le + brk;
        line_no++;
        bool blank = true;
        for (const unsigned char *c = b; c < le;) {
            const int n = space_len(c, le);
            if (!n) { blank = false; break; }
            c += n;
        }
        if (blank) continue;
        P.reset((const char *)b, (const char *)le);
        if (le - b >= 3 && b[0] == 0xEF && b[1] == 0xBB && b[2] == 0xBF)
            return err(RSIM_IO_JSON, "invalid JSON: Unexpected UTF-8 BOM (decode using utf-8-sig)");
        Val top;
        P.ws();
        bool ok = P.value(top, 0, false);
        if (ok) { P.ws(); if (P.p != P.e) ok = P.fail("Extra data"); }
        if (!ok) return err(RSIM_IO_JSON, "invalid JSON: " + P.msg);
        if (top.k != K_OBJ) return err(RSIM_IO_RECORD, "record is not an object");
        const char *req[5] = {"id", "arrival_s", "blocks", "in", "out"};
        const bool have[5] = {P.id.k != K_NONE, P.arr.k != K_NONE, P.has_blocks, P.in.k != K_NONE, P.out.k != K_NONE};
        for (int f = 0; f < 5; f++)
            if (!have[f]) return err(RSIM_IO_RECORD, std::string("missing field '") + req[f] + "'");
        auto is_int = [](const Val &v) { return v.k == K_INT || v.k == K_BOOL || v.k == K_NEGINT || v.k == K_BIGINT; };
        if (!is_int(P.id) || P.id.k == K_NEGINT) return err(RSIM_IO_RECORD, "id must be a non-negative integer");
        const double a = P.arr.num();
        if (!((P.arr.k == K_INT || P.arr.k == K_NEGINT || P.arr.k == K_BIGINT || P.arr.k == K_FLOAT) && !(a < 0)))
            return err(RSIM_IO_RECORD, "arrival_s must be a non-negative number");
        if (P.blocks.k != K_ARR || P.bv.empty()) return err(RSIM_IO_RECORD, "blocks must be a non-empty list");
        if (!P.blocks_ok) return err(RSIM_IO_RECORD, "block hashes must be u64");
        if (!is_int(P.in) || P.in.k == K_NEGINT || (P.in.k != K_BIGINT && P.in.u < 1))
            return err(RSIM_IO_RECORD, "in must be a positive integer");
        if (!is_int(P.out) || P.out.k == K_NEGINT || (P.out.k != K_BIGINT && P.out.u < 1))
            return err(RSIM_IO_RECORD, "out must be a positive integer");
        uint64_t ck;
        if (P.cls.k == K_NONE || P.cls.k == K_NULL) ck = class_key2(P.bv.data(), P.bv.size());
        else if (P.cls.k == K_INT || P.cls.k == K_BOOL) ck = P.cls.u;
        else return err(RSIM_IO_RECORD, "class must be u64");
        if (P.id.k == K_BIGINT) return err(RSIM_IO_UNSUPPORTED, "id does not fit in 64 bits (packed trace)");
        if (P.in.k == K_BIGINT || P.out.k == K_BIGINT || P.in.u > (uint64_t)INT64_MAX || P.out.u > (uint64_t)INT64_MAX)
            return err(RSIM_IO_UNSUPPORTED, "in/out do not fit in 63 bits (packed trace)");
        if (a < prev) {                                   // load_trace, trace.py:160-164
            R->arrival = a; R->previous = prev;
            return err(RSIM_IO_ORDER, "arrival before previous");
        }
        prev = a;
        R->id.push_back(P.id.u); R->arr.push_back(a); R->in.push_back((int64_t)P.in.u);
        R->out.push_back((int64_t)P.out.u); R->cls.push_back(ck);
        R->blocks.insert(R->blocks.end(), P.bv.begin(), P.bv.end());
        R->off.push_back((int64_t)R->blocks.size());
    }
    return RSIM_IO_OK;
}

int rsim_trace_parse_status(const rsim_trace_parse *p) { return p ? p->status : RSIM_IO_JSON; }

int64_t rsim_trace_parse_count(const rsim_trace_parse *p, int64_t *n_blocks) {
    if (n_blocks) *n_blocks = (int64_t)p->blocks.size();
    return (int64_t)p->id.size();
}

void rsim_trace_parse_copy(const rsim_trace_parse *p, uint64_t *request_id, double *arrival_s, int64_t *in_tokens,
                           int64_t *out_tokens, uint64_t *class_key, int64_t *blk_off, uint64_t *blocks) {
    const size_t n = p->id.size();
    if (request_id) memcpy(request_id, p->id.data(), n * sizeof(uint64_t));
    if (arrival_s) memcpy(arrival_s, p->arr.data(), n * sizeof(double));
    if (in_tokens) memcpy(in_tokens, p->in.data(), n * sizeof(int64_t));
    if (out_tokens) memcpy(out_tokens, p->out.data(), n * sizeof(int64_t));
    if (class_key) memcpy(class_key, p->cls.data(), n * sizeof(uint64_t));
    if (blk_off) memcpy(blk_off, p->off.data(), (n + 1) * sizeof(int64_t));
    if (blocks) memcpy(blocks, p->blocks.data(), p->blocks.size() * sizeof(uint64_t));
}

const char *rsim_trace_parse_error(const rsim_trace_parse *p, int64_t *line, double *arrival, double *previous) {
    if (line) *line = p->line;
    if (arrival) *arrival = p->arrival;
    if (previous) *previous = p->previous;
    return p->msg.c_str();
}

void rsim_trace_parse_free(rsim_trace_parse *p) { delete p; }

}  // extern "C"
