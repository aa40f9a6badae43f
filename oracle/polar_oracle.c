/* TEST INFRASTRUCTURE ONLY — plain-C CPU oracle for the polar decoder path.
 *
 * Restates the reference's FrameDecoder<R>::decode path
 * (/root/reference/proj/include/polar/decoders.hpp:60-85) and everything it
 * calls: the decode tree (prune_tree.cpp:38-71, prune_tree.hpp:78-105), the
 * CRC engine (crc.cpp:86-154), the SC decoder (sc_decoder.hpp) and the list
 * decoder in its copy layout (list_decoder.hpp).  The precision-generic part
 * lives in oracle_core.inc.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load this library, and only as the checker.
 *
 * Parity pinned against the unmodified reference (oracle/_ref, built by
 * oracle/Makefile) and the golden vectors in tests/golden/.
 */
#define _POSIX_C_SOURCE 200809L
#include "polar_oracle.h"

#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* NodeKind (prune_tree.hpp:11-19), same numbering */
enum { NK_BRANCH, NK_FROZEN, NK_INFO, NK_R0, NK_R1, NK_REP, NK_SPC };

/* ApplyKind (list_decoder.hpp:102) */
enum { AK_BIT, AK_BCAST, AK_FLIPS };

typedef struct {
    int kind, depth, leaf_begin, size, left, right;
} orc_node;

typedef struct {
    int n, stages, count;
    orc_node* nodes;
} orc_tree_t;

typedef struct {
    int n, k, crc_width, reflect;
    uint64_t poly, init, xorout;
    uint64_t table[256];
    uint64_t rpoly, poly_top, init_reg;
    const uint8_t* frozen;
} orc_code;

typedef struct {
    uint8_t* codeword;
    int crc_ok, esc;
    double metric;
} orc_result;

/* ---- decode tree: prune_tree.cpp:38-71 -------------------------------- */

static int tree_build(orc_tree_t* t, const uint8_t* frozen, int lo, int size, int depth,
                      const int32_t* pc) {
    int idx = t->count++;
    orc_node* nd = &t->nodes[idx];
    nd->depth = depth;
    nd->leaf_begin = lo;
    nd->size = size;
    nd->left = nd->right = -1;
    int nfrozen = 0;
    for (int i = 0; i < size; ++i) nfrozen += frozen[lo + i] != 0;
    int kind = NK_BRANCH;
    if (size == 1) {
        kind = nfrozen ? NK_FROZEN : NK_INFO;
    } else if (pc[2] && nfrozen == size - 1 && !frozen[lo + size - 1] &&
               (pc[4] == 0 || size <= pc[4])) {
        kind = NK_REP;
    } else if (pc[3] && nfrozen == 1 && frozen[lo] && (pc[5] == 0 || size <= pc[5])) {
        kind = NK_SPC;
    } else if (pc[0] && nfrozen == size) {
        kind = NK_R0;
    } else if (pc[1] && nfrozen == 0) {
        kind = NK_R1;
    }
    nd->kind = kind;
    if (kind == NK_BRANCH && size > 1) {
        int l = tree_build(t, frozen, lo, size / 2, depth + 1, pc);
        int r = tree_build(t, frozen, lo + size / 2, size / 2, depth + 1, pc);
        t->nodes[idx].left = l;
        t->nodes[idx].right = r;
    }
    return idx;
}

/* prune_tree.cpp:24-35 validation; returns 0 on success */
static int tree_init(orc_tree_t* t, const uint8_t* frozen, int n, const int32_t* pc) {
    if (n < 2 || (n & (n - 1)) != 0) return 1;
    if (pc[4] < 0 || pc[5] < 0 || (pc[4] && pc[4] < 2) || (pc[5] && pc[5] < 4)) return 1;
    t->n = n;
    t->stages = 0;
    while ((1 << t->stages) < n) ++t->stages;
    t->count = 0;
    t->nodes = calloc((size_t)(2 * n), sizeof(orc_node));
    if (!t->nodes) return 1;
    tree_build(t, frozen, 0, n, 0, pc);
    return 0;
}

/* ---- CRC engine: crc.cpp:86-154 ---------------------------------------- */

static uint64_t bit_rev(uint64_t v, int w) {
    uint64_t r = 0;
    for (int i = 0; i < w; ++i) {
        r = (r << 1) | (v & 1);
        v >>= 1;
    }
    return r;
}

static void crc_init(orc_code* c) {
    if (c->reflect) {
        c->rpoly = bit_rev(c->poly, c->crc_width);
        c->init_reg = bit_rev(c->init, c->crc_width);
        for (int b = 0; b < 256; ++b) {
            uint64_t r = (uint64_t)b;
            for (int i = 0; i < 8; ++i) r = (r >> 1) ^ ((r & 1) ? c->rpoly : 0);
            c->table[b] = r;
        }
    } else {
        c->poly_top = c->poly << (64 - c->crc_width);
        c->init_reg = c->init << (64 - c->crc_width);
        for (int b = 0; b < 256; ++b) {
            uint64_t r = (uint64_t)b << 56;
            for (int i = 0; i < 8; ++i) {
                int top = (int)(r >> 63);
                r <<= 1;
                if (top) r ^= c->poly_top;
            }
            c->table[b] = r;
        }
    }
}

/* crc.cpp:121-144 over bits given one per byte */
static uint64_t crc_compute(const orc_code* c, const uint8_t* bits, size_t len) {
    uint64_t reg = c->init_reg;
    size_t nbytes = len / 8;
    if (c->reflect) {
        for (size_t k = 0; k < nbytes; ++k) {
            unsigned byte = 0;
            for (int j = 0; j < 8; ++j) byte = (byte << 1) | (bits[8 * k + j] & 1u);
            reg = (reg >> 8) ^ c->table[(reg ^ byte) & 0xFF];
        }
        for (size_t i = nbytes * 8; i < len; ++i) {
            reg ^= (uint64_t)(bits[i] & 1u);
            int lo = (int)(reg & 1);
            reg >>= 1;
            if (lo) reg ^= c->rpoly;
        }
        return reg ^ c->xorout;
    }
    for (size_t k = 0; k < nbytes; ++k) {
        unsigned byte = 0;
        for (int j = 0; j < 8; ++j) byte = (byte << 1) | (bits[8 * k + j] & 1u);
        reg = (reg << 8) ^ c->table[((reg >> 56) ^ byte) & 0xFF];
    }
    for (size_t i = nbytes * 8; i < len; ++i) {
        reg ^= (uint64_t)(bits[i] & 1u) << 63;
        int top = (int)(reg >> 63);
        reg <<= 1;
        if (top) reg ^= c->poly_top;
    }
    return (reg >> (64 - c->crc_width)) ^ c->xorout;
}

/* prune_tree.hpp:78-105 — the payload is the decision word gathered at the
 * open positions in ascending order (test_tree.cpp:125-146 pins this
 * equivalence), then crc.cpp:146-154 checks it. */
static int orc_payload_crc_ok(const orc_code* c, const orc_tree_t* t, const uint8_t* word) {
    (void)t;
    int psize = c->k + c->crc_width;
    uint8_t stackbuf[4096];
    uint8_t* pay = psize <= 4096 ? stackbuf : malloc((size_t)psize);
    int w = 0;
    for (int i = 0; i < c->n; ++i)
        if (!c->frozen[i]) pay[w++] = word[i];
    size_t len = (size_t)(psize - c->crc_width);
    uint64_t tail = 0;
    for (int j = 0; j < c->crc_width; ++j) tail = (tail << 1) | pay[len + (size_t)j];
    int ok = crc_compute(c, pay, len) == tail;
    if (pay != stackbuf) free(pay);
    return ok;
}

/* ---- precision-generic core ------------------------------------------- */

#define R float
#define SFX(x) x##_f32
#define RFIX 0
#include "oracle_core.inc"
#undef R
#undef SFX
#undef RFIX

#define R int8_t
#define SFX(x) x##_i8
#define RFIX 1
#define RMAX 127
#include "oracle_core.inc"
#undef R
#undef SFX
#undef RFIX
#undef RMAX

/* ---- decoder object ---------------------------------------------------- */

struct orc_decoder {
    orc_code code;
    uint8_t* frozen;
    orc_tree_t tree;
    int kind, l, precision;
};

static void set_err(char* err, int errlen, const char* msg) {
    if (err && errlen > 0) snprintf(err, (size_t)errlen, "%s", msg);
}

static int uses_list(int kind) { return kind >= 2; }
static int uses_crc(int kind) { return kind >= 4; }
static int adaptive(int kind) { return kind >= 5; }
static int uses_pruning(int kind) { return kind != 0 && kind != 2; }

orc_decoder* orc_create(int n, int k, const uint8_t* frozen, int crc_width,
                        uint64_t poly, int reflect, uint64_t init, uint64_t xorout,
                        int kind, int l, int precision, const int32_t* pruning,
                        char* err, int errlen) {
    static const int32_t none[6] = {0, 0, 0, 0, 0, 0};
    if (n < 2 || (n & (n - 1)) != 0) { set_err(err, errlen, "N must be a power of two >= 2"); return NULL; }
    if (k < 1) { set_err(err, errlen, "K must be at least 1"); return NULL; }
    if (kind < 0 || kind > 6 || precision < 0 || precision > 1) { set_err(err, errlen, "bad kind/precision"); return NULL; }
    if (crc_width < 0 || crc_width > 64) { set_err(err, errlen, "CRC width must be in [1, 64]"); return NULL; }
    if (crc_width) {
        uint64_t mask = crc_width == 64 ? ~0ull : ((1ull << crc_width) - 1);
        if ((poly & ~mask) || (init & ~mask) || (xorout & ~mask) || !(poly & 1)) {
            set_err(err, errlen, "bad CRC spec");
            return NULL;
        }
    }
    int open = 0;
    for (int i = 0; i < n; ++i) open += frozen[i] == 0;
    if (open != k + crc_width) { set_err(err, errlen, "frozen mask does not leave K + CRC open positions"); return NULL; }
    int ll = uses_list(kind) ? l : 1;
    if (uses_crc(kind) && !crc_width) { set_err(err, errlen, "CRC-aided decoding needs a code with a CRC"); return NULL; }
    if (adaptive(kind) && ll < 2) { set_err(err, errlen, "adaptive decoding needs a list limit of at least 2"); return NULL; }
    if (uses_list(kind) && (ll < 1 || (ll & (ll - 1)) != 0)) { set_err(err, errlen, "list size must be a power of two"); return NULL; }

    orc_decoder* d = calloc(1, sizeof(*d));
    d->frozen = malloc((size_t)n);
    memcpy(d->frozen, frozen, (size_t)n);
    d->code.n = n;
    d->code.k = k;
    d->code.crc_width = crc_width;
    d->code.poly = poly;
    d->code.reflect = reflect;
    d->code.init = init;
    d->code.xorout = xorout;
    d->code.frozen = d->frozen;
    if (crc_width) crc_init(&d->code);
    if (tree_init(&d->tree, d->frozen, n, uses_pruning(kind) ? pruning : none)) {
        set_err(err, errlen, "bad pruning caps");
        free(d->frozen);
        free(d);
        return NULL;
    }
    d->kind = kind;
    d->l = ll;
    d->precision = precision;
    return d;
}

void orc_destroy(orc_decoder* d) {
    if (!d) return;
    free(d->tree.nodes);
    free(d->frozen);
    free(d);
}

static void pack_msb(const uint8_t* bits, int nbits, uint8_t* out) {
    memset(out, 0, (size_t)(nbits + 7) / 8);
    for (int i = 0; i < nbits; ++i)
        if (bits[i]) out[i >> 3] |= (uint8_t)(0x80u >> (i & 7));
}

static void emit(const orc_decoder* d, const uint8_t* cw, int64_t f, uint8_t* payload,
                 uint8_t* codeword) {
    int n = d->code.n, psize = d->code.k + d->code.crc_width;
    if (codeword) pack_msb(cw, n, codeword + (size_t)f * (size_t)((n + 7) / 8));
    if (payload) {
        uint8_t* out = payload + (size_t)f * (size_t)((psize + 7) / 8);
        memset(out, 0, (size_t)(psize + 7) / 8);
        int w = 0;
        for (int i = 0; i < n; ++i)
            if (!d->frozen[i]) {
                if (cw[i]) out[w >> 3] |= (uint8_t)(0x80u >> (w & 7));
                ++w;
            }
    }
}

typedef struct {
    const orc_decoder* d;
    const void* llr;
    int64_t f0, f1;
    uint8_t *payload, *codeword, *crc_ok, *esc;
    double* metric;
} job_t;

static void* run_job(void* arg) {
    job_t* j = arg;
    const orc_decoder* d = j->d;
    int n = d->code.n;
    uint8_t* cw = malloc((size_t)n);
    orc_result res = {cw, 0, 1, 0.0};
    if (d->precision == 0) {
        sc_state_f32 sc = {&d->tree, calloc(2 * (size_t)n, sizeof(float)), calloc((size_t)n, 1),
                           calloc((size_t)n, sizeof(float))};
        list_state_f32 ls;
        list_alloc_f32(&ls, &d->tree, d->l);
        for (int64_t f = j->f0; f < j->f1; ++f) {
            frame_decode_f32(&sc, &ls, &d->code, d->kind, d->l,
                             (const float*)j->llr + (size_t)f * (size_t)n, &res);
            emit(d, cw, f, j->payload, j->codeword);
            if (j->crc_ok) j->crc_ok[f] = (uint8_t)res.crc_ok;
            if (j->esc) j->esc[f] = (uint8_t)res.esc;
            if (j->metric) j->metric[f] = res.metric;
        }
        list_free_f32(&ls);
        free(sc.llr); free(sc.ps); free(sc.fold);
    } else {
        sc_state_i8 sc = {&d->tree, calloc(2 * (size_t)n, 1), calloc((size_t)n, 1),
                          calloc((size_t)n, 1)};
        list_state_i8 ls;
        list_alloc_i8(&ls, &d->tree, d->l);
        for (int64_t f = j->f0; f < j->f1; ++f) {
            frame_decode_i8(&sc, &ls, &d->code, d->kind, d->l,
                            (const int8_t*)j->llr + (size_t)f * (size_t)n, &res);
            emit(d, cw, f, j->payload, j->codeword);
            if (j->crc_ok) j->crc_ok[f] = (uint8_t)res.crc_ok;
            if (j->esc) j->esc[f] = (uint8_t)res.esc;
            if (j->metric) j->metric[f] = res.metric;
        }
        list_free_i8(&ls);
        free(sc.llr); free(sc.ps); free(sc.fold);
    }
    free(cw);
    return NULL;
}

int orc_decode(orc_decoder* d, const void* llr, int64_t nframes, int nthreads,
               uint8_t* payload, uint8_t* codeword, uint8_t* crc_ok, uint8_t* esc,
               double* metric) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > nframes) nthreads = (int)(nframes > 0 ? nframes : 1);
    job_t* jobs = calloc((size_t)nthreads, sizeof(job_t));
    pthread_t* th = calloc((size_t)nthreads, sizeof(pthread_t));
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = (job_t){d, llr, nframes * t / nthreads, nframes * (t + 1) / nthreads,
                          payload, codeword, crc_ok, esc, metric};
        if (nthreads == 1) run_job(&jobs[t]);
        else pthread_create(&th[t], NULL, run_job, &jobs[t]);
    }
    if (nthreads > 1)
        for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(jobs);
    free(th);
    return 0;
}

int orc_list_decode(orc_decoder* d, const void* llr, int l, int select_by_crc,
                    uint8_t* payload, uint8_t* codeword, uint8_t* crc_ok,
                    double* metric, uint8_t* alive, double* slot_metric) {
    if (!uses_list(d->kind) || l < 1 || l > d->l || (l & (l - 1))) return 1;
    if (select_by_crc && !d->code.crc_width) return 1;
    int n = d->code.n;
    uint8_t* cw = malloc((size_t)n);
    orc_result res = {cw, 0, 1, 0.0};
    if (d->precision == 0) {
        list_state_f32 ls;
        list_alloc_f32(&ls, &d->tree, d->l);
        list_decode_f32(&ls, &d->code, (const float*)llr, l, select_by_crc, &res);
        for (int p = 0; p < d->l; ++p) {
            alive[p] = ls.alive[p];
            slot_metric[p] = ls.alive[p] ? (double)ls.metric[p] : 0.0;
        }
        list_free_f32(&ls);
    } else {
        list_state_i8 ls;
        list_alloc_i8(&ls, &d->tree, d->l);
        list_decode_i8(&ls, &d->code, (const int8_t*)llr, l, select_by_crc, &res);
        for (int p = 0; p < d->l; ++p) {
            alive[p] = ls.alive[p];
            slot_metric[p] = ls.alive[p] ? (double)ls.metric[p] : 0.0;
        }
        list_free_i8(&ls);
    }
    emit(d, cw, 0, payload, codeword);
    *crc_ok = (uint8_t)res.crc_ok;
    *metric = res.metric;
    free(cw);
    return 0;
}

int orc_tree(const uint8_t* frozen, int n, const int32_t* pruning, int32_t* out,
             int max_nodes) {
    orc_tree_t t;
    if (tree_init(&t, frozen, n, pruning)) return -1;
    if (t.count > max_nodes) {
        free(t.nodes);
        return -1;
    }
    for (int i = 0; i < t.count; ++i) {
        const orc_node* nd = &t.nodes[i];
        out[6 * i + 0] = nd->kind;
        out[6 * i + 1] = nd->depth;
        out[6 * i + 2] = nd->leaf_begin;
        out[6 * i + 3] = nd->size;
        out[6 * i + 4] = nd->left;
        out[6 * i + 5] = nd->right;
    }
    int cnt = t.count;
    free(t.nodes);
    return cnt;
}

void orc_kernels_f32(float a, float b, float* out) {
    out[0] = fk_f32(a, b);
    out[1] = gk_f32(a, b, 0);
    out[2] = gk_f32(a, b, 1);
    out[3] = sat_add_f32(a, b);
    out[4] = (float)hard_f32(a);
}

void orc_kernels_i8(int a, int b, int* out) {
    out[0] = fk_i8((int8_t)a, (int8_t)b);
    out[1] = gk_i8((int8_t)a, (int8_t)b, 0);
    out[2] = gk_i8((int8_t)a, (int8_t)b, 1);
    out[3] = sat_add_i8((int8_t)a, (int8_t)b);
    out[4] = hard_i8((int8_t)a);
}

void orc_two_smallest_f32(const float* v, int n, int* i1, int* i2) {
    two_smallest_f32(v, n, i1, i2);
}

uint64_t orc_crc(int width, uint64_t poly, int reflect, uint64_t init,
                 uint64_t xorout, const uint8_t* bits, int64_t len) {
    orc_code c;
    memset(&c, 0, sizeof(c));
    c.crc_width = width;
    c.poly = poly;
    c.reflect = reflect;
    c.init = init;
    c.xorout = xorout;
    crc_init(&c);
    return crc_compute(&c, bits, (size_t)len);
}
