/*
 * lgreco_ref.c -- CPU ORACLE for the L-GreCo data-parallel hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2210_17357_b200/) never links, imports or calls it.
 * It shares no code, header, table or constant generator with the CUDA path.
 *
 * Plain, slow, obviously-correct scalar C.  Build:
 *   gcc -O2 -ffp-contract=off -fno-fast-math -fPIC -shared -o liblgreco_ref.so lgreco_ref.c -lm
 * (no FMA contraction except the explicit fmaf() the pinned quantiser uses; no FTZ).
 *
 * Citations (PAPER.md = /root/reference/PAPER.md, L-GreCo, MLSys'23):
 *   Metric: L2 norm of the error of a simulated compress->decompress, "without
 *     applying error feedback"             PAPER.md:171-183, 191, 313-314 (§3, §4)
 *   Problem: min sum size s.t. sum error <= Emax      PAPER.md:185-200 (§3 eqn)
 *   Emax from the uniform default                       PAPER.md:206-210; Alg.1 l.2
 *   Discretisation D=10000, step Emax/D                 PAPER.md:251-255; Alg.1 l.3-5
 *   Algorithm 1 DP + backtracking
 *   Compressors: quantisation / TopK / PowerSGD, EF
 * Where the paper is silent the readings are those of SURVEY.md §8(c), listed in
 * DESIGN.md "Readings" (R1..R20); each function names the readings it uses.
 *
 * Parity status: every function below is pinned by tests/test_oracle_*.py
 * (KATs, closed forms, brute force, textbook identities); none is "parity unpinned".
 */
#include <math.h>
#include <float.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define REF_OK 0
#define REF_EINVAL (-1)
#define REF_ENONFINITE (-2)
#define REF_EINFEASIBLE (-3)
#define REF_ENOMEM (-6)

typedef struct {
    int64_t offset, numel;
    int32_t rows, cols, compress;
} ref_layer;

typedef struct {
    double emax, total_err;
    int64_t total_bits, default_bits;
    int32_t used_default, n_active;
} ref_solve_info;

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon et al., SC'11; Random123 constants).  Reading R3.    */
/* ------------------------------------------------------------------------ */
static void philox_round(uint32_t c[4], const uint32_t k[2]) {
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c[0];
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c[1] ^ k[0];
    uint32_t n2 = hi0 ^ c[3] ^ k[1];
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
}

void ref_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
    uint32_t k[2] = {key[0], key[1]};
    for (int r = 0; r < 10; r++) {
        if (r > 0) { k[0] += 0x9E3779B9u; k[1] += 0xBB67AE85u; }
        philox_round(c, k);
    }
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

/* u in [0,1): 24 high bits of the Philox word (R3). */
static float word_to_u(uint32_t w) { return (float)(w >> 8) * 5.9604644775390625e-08f; }

/* One uniform: word `w` of Philox(ctr=(c0, rankfield, step_lo32, stream)) (R3). */
float ref_uniform(uint64_t seed, uint32_t rankfield, uint64_t step, uint32_t stream,
                  uint32_t c0, int32_t w) {
    uint32_t ctr[4] = {c0, rankfield, (uint32_t)step, stream};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t o[4];
    ref_philox4x32_10(ctr, key, o);
    return word_to_u(o[w & 3]);
}

/* Fill u[0..nvalid) for bucket gb of quant bucket size B (R3):
 * element p uses ctr=(gb*(B/4) + p/4, rankfield, step_lo32, stream), word p%4. */
void ref_bucket_uniforms(uint64_t seed, uint32_t rankfield, uint64_t step, uint32_t stream,
                         int64_t gb, int32_t B, int32_t nvalid, float* u) {
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    for (int p = 0; p < nvalid; p++) {
        uint32_t ctr[4] = {(uint32_t)((uint64_t)gb * (uint64_t)(B / 4) + (uint64_t)(p / 4)),
                           rankfield, (uint32_t)step, stream};
        uint32_t o[4];
        ref_philox4x32_10(ctr, key, o);
        u[p] = word_to_u(o[p % 4]);
    }
}

/* x = fl(fl(g + e) + 0): gradient plus error feedback, -0 canonicalised to +0 (R2). */
static float canon_x(float g, const float* e, int64_t i) {
    volatile float s = (e ? g + e[i] : g);
    return s + 0.0f;
}

/* ------------------------------------------------------------------------ */
/* Paper-mode accumulation (row a1): "we accumulate per-layer    */
/* gradients in auxiliary buffers"; G <- G + g, one fp32 add per element.     */
/* ------------------------------------------------------------------------ */
void ref_accumulate(float* G, const float* g, int64_t n) {
    for (int64_t i = 0; i < n; i++) {
        volatile float s = G[i] + g[i];
        G[i] = s;
    }
}

/* ------------------------------------------------------------------------ */
/* QSGD-style bucketed min/max stochastic quantiser (R5, R6).                */
/* ------------------------------------------------------------------------ */
/* Quantise one bucket of nvalid values with `bits` bits using the uniforms u.
 * Writes codes q[], decoded dec[], and metadata (mn, unit).  Returns status. */
int ref_quantize_bucket(const float* x, int32_t nvalid, int32_t bits, const float* u,
                        uint32_t* q, float* dec, float* mn_out, float* unit_out) {
    if (bits < 1 || bits > 16 || nvalid <= 0) return REF_EINVAL;
    for (int i = 0; i < nvalid; i++)
        if (!isfinite(x[i])) return REF_ENONFINITE;
    float mn = x[0], mx = x[0];
    for (int i = 1; i < nvalid; i++) {
        if (x[i] < mn) mn = x[i];
        if (x[i] > mx) mx = x[i];
    }
    float s = (float)((1u << bits) - 1u);
    float unit = 0.0f;
    int constant = (mx == mn);
    if (!constant) {
        float range = mx - mn;
        if (isinf(range)) return REF_ENONFINITE;
        /* inv = RD(s / range), the largest float <= s / range (R5): from the IEEE RN
         * quotient, stepped down when it lies above (the float products are exact in
         * double).  Then t * inv <= s for every t <= range, so q <= s. */
        float inv = s / range;
        if (isfinite(inv) && (double)inv * (double)range > (double)s) inv = nextafterf(inv, 0.0f);
        unit = range / s;
        if (!(inv < FLT_MAX)) {
            constant = 1; /* near-subnormal range (s / range >= FLT_MAX): treated as constant, unit kept */
        } else {
            for (int i = 0; i < nvalid; i++) {
                float t = x[i] - mn;
                /* v = t * inv taken exactly: the product of two floats has at most
                 * 48 significant bits, so the double product is exact (R6). */
                double v = (double)t * (double)inv;
                double fl = floor(v);
                double f = v - fl; /* exact: v and fl share the exponent range */
                double qq = fl + (((double)u[i] < f) ? 1.0 : 0.0);
                if (qq > (double)s) qq = (double)s;
                q[i] = (uint32_t)qq;
                dec[i] = fmaf((float)qq, unit, mn);
            }
        }
    }
    if (constant) {
        for (int i = 0; i < nvalid; i++) { q[i] = 0u; dec[i] = fmaf(0.0f, unit, mn); }
    }
    *mn_out = mn;
    *unit_out = unit;
    return REF_OK;
}

/* ------------------------------------------------------------------------ */
/* Payload layout (R7): records in global bucket order.                       */
/*   compressed layer, b bits, bucket B=128m: (4*b*m) u32 code words, mn, unit */
/*     word (t*b + p)*4 + s, bit l  <-  bit p of code of element 128t+4l+s     */
/*   lossless layer: records of B raw fp32 values (last one partial)           */
/*   each layer's block of records starts at a 16-byte boundary (zero pad)    */
/* ------------------------------------------------------------------------ */
static int64_t nbuckets(int64_t n, int32_t B) { return (n + B - 1) / B; }

static int64_t rec_bytes_full(int32_t lbits, int32_t B) {
    return lbits > 0 ? (int64_t)16 * lbits * (B / 128) + 8 : (int64_t)4 * B;
}

/* Per-layer layout: bucket_start[L+1], byte_off[L+1]; returns total bytes. */
int64_t ref_layout(const ref_layer* layers, int32_t L, const int32_t* lbits, int32_t B,
                   int64_t* bucket_start, int64_t* byte_off) {
    int64_t gb = 0, off = 0;
    for (int l = 0; l < L; l++) {
        bucket_start[l] = gb;
        byte_off[l] = off;
        int64_t nb = nbuckets(layers[l].numel, B);
        gb += nb;
        off += lbits[l] > 0 ? nb * rec_bytes_full(lbits[l], B) : 4 * layers[l].numel;
        off = (off + 15) & ~(int64_t)15; /* each layer's records start 16-byte aligned (R7) */
    }
    bucket_start[L] = gb;
    byte_off[L] = off;
    return off;
}

static void pack_record(uint8_t* dst, const uint32_t* q, int32_t nvalid, int32_t bits, int32_t B,
                        float mn, float unit) {
    int m = B / 128;
    uint32_t tmp[4 * 16 * 64];
    memset(tmp, 0, sizeof(uint32_t) * 4 * bits * m);
    for (int e = 0; e < nvalid; e++) {
        int t = e / 128, r = e % 128, l = r / 4, s = r % 4;
        for (int p = 0; p < bits; p++)
            if ((q[e] >> p) & 1u) tmp[(t * bits + p) * 4 + s] |= (1u << l);
    }
    memcpy(dst, tmp, sizeof(uint32_t) * 4 * bits * m);
    memcpy(dst + 16 * bits * m, &mn, 4);
    memcpy(dst + 16 * bits * m + 4, &unit, 4);
}

static void unpack_record(const uint8_t* src, int32_t nvalid, int32_t bits, int32_t B, float* out) {
    int m = B / 128;
    uint32_t tmp[4 * 16 * 64];
    float mn, unit;
    memcpy(tmp, src, sizeof(uint32_t) * 4 * bits * m);
    memcpy(&mn, src + 16 * bits * m, 4);
    memcpy(&unit, src + 16 * bits * m + 4, 4);
    for (int e = 0; e < nvalid; e++) {
        int t = e / 128, r = e % 128, l = r / 4, s = r % 4;
        uint32_t q = 0;
        for (int p = 0; p < bits; p++) q |= ((tmp[(t * bits + p) * 4 + s] >> l) & 1u) << p;
        out[e] = fmaf((float)q, unit, mn);
    }
}

/* Quantise one layer's values xs (canonical) into records starting at pay (stage
 * `stream`, rank field `rankfield`); dec receives decoded values. */
static int quantize_layer(const float* xs, int64_t n, int32_t bits, int32_t B, int64_t gb0,
                          uint64_t seed, uint32_t rankfield, uint64_t step, uint32_t stream,
                          uint8_t* pay, float* dec) {
    float* u = (float*)malloc(sizeof(float) * B);
    uint32_t* q = (uint32_t*)malloc(sizeof(uint32_t) * B);
    if (!u || !q) { free(u); free(q); return REF_ENOMEM; }
    int64_t nb = nbuckets(n, B);
    int st = REF_OK;
    for (int64_t j = 0; j < nb && st == REF_OK; j++) {
        int32_t nv = (int32_t)((n - j * B) < B ? (n - j * B) : B);
        float mn, unit;
        ref_bucket_uniforms(seed, rankfield, step, stream, gb0 + j, B, nv, u);
        st = ref_quantize_bucket(xs + j * B, nv, bits, u, q, dec + j * B, &mn, &unit);
        if (st == REF_OK && pay) pack_record(pay + j * rec_bytes_full(bits, B), q, nv, bits, B, mn, unit);
    }
    free(u); free(q);
    return st;
}

/* QSGD profile (a2): err[l][j] = ||x_l - Q_{b_j}(x_l)||_2 (fp64), stage-1 uniforms,
 * EF not updated; bits[l][j] = ceil(n/B)*(B*b+64).
 * Lossless layers get err 0, bits 32n for every candidate.                  */
int ref_qsgd_profile(const ref_layer* layers, int32_t L, const float* g, const float* e,
                     const int32_t* cand_bits, int32_t K, int32_t B, uint64_t seed,
                     uint32_t rank, uint64_t step, double* err, int64_t* bits) {
    if (B <= 0 || B % 128 || B > 8192) return REF_EINVAL;
    /* first global bucket of every layer (the Philox counter base) */
    int64_t* gb0 = (int64_t*)malloc(sizeof(int64_t) * (size_t)(L + 1));
    if (!gb0) return REF_ENOMEM;
    gb0[0] = 0;
    for (int l = 0; l < L; l++) gb0[l + 1] = gb0[l] + nbuckets(layers[l].numel, B);
    int status = REF_OK;
    /* layers are independent: with -fopenmp (the oracle's OpenMP build, a timing
     * baseline only) they run on all host cores; the arithmetic of each is unchanged */
#pragma omp parallel for schedule(dynamic, 1)
    for (int l = 0; l < L; l++) {
        int64_t n = layers[l].numel, nb = nbuckets(n, B), gb = gb0[l];
        if (!layers[l].compress) {
            for (int j = 0; j < K; j++) { err[l * K + j] = 0.0; bits[l * K + j] = 32 * n; }
            continue;
        }
        float* xs = (float*)malloc(sizeof(float) * (size_t)n);
        float* dec = (float*)malloc(sizeof(float) * (size_t)n);
        if (!xs || !dec) {
            free(xs); free(dec);
#pragma omp critical
            status = REF_ENOMEM;
            continue;
        }
        for (int64_t i = 0; i < n; i++) xs[i] = canon_x(g[layers[l].offset + i], e ? e + layers[l].offset : NULL, i);
        for (int j = 0; j < K; j++) {
            int st = quantize_layer(xs, n, cand_bits[j], B, gb, seed, rank, step, 0u, NULL, dec);
            if (st) {
#pragma omp critical
                status = st;
                break;
            }
            double sse = 0.0;
            for (int64_t i = 0; i < n; i++) {
                double d = (double)xs[i] - (double)dec[i];
                sse += d * d;
            }
            err[l * K + j] = sqrt(sse);
            bits[l * K + j] = nb * ((int64_t)B * cand_bits[j] + 64);
        }
        free(xs); free(dec);
    }
    free(gb0);
    return status;
}

/* Stage-1 compress of one rank (a8): x = g+e; pack with lbits[l] (0 = lossless);
 * e <- x - dec (R15); dec_out (nullable) receives dec.                      */
int ref_qsgd_pack(const ref_layer* layers, int32_t L, const int32_t* lbits, int32_t B,
                  uint64_t seed, uint32_t rank, uint64_t step, const float* g, float* e,
                  uint8_t* payload, float* dec_out) {
    int64_t* bs = (int64_t*)malloc(sizeof(int64_t) * (L + 1));
    int64_t* bo = (int64_t*)malloc(sizeof(int64_t) * (L + 1));
    ref_layout(layers, L, lbits, B, bs, bo);
    int status = REF_OK;
    /* layers are independent (own records, own EF range): OpenMP build only */
#pragma omp parallel for schedule(dynamic, 1)
    for (int l = 0; l < L; l++) {
        int64_t n = layers[l].numel, o = layers[l].offset;
        int st = REF_OK;
        float* xs = (float*)malloc(sizeof(float) * (size_t)n);
        float* dec = (float*)malloc(sizeof(float) * (size_t)n);
        for (int64_t i = 0; i < n; i++) xs[i] = canon_x(g[o + i], e ? e + o : NULL, i);
        if (lbits[l] > 0) {
            st = quantize_layer(xs, n, lbits[l], B, bs[l], seed, rank, step, 0u, payload + bo[l], dec);
        } else {
            memcpy(payload + bo[l], xs, sizeof(float) * (size_t)n);
            memcpy(dec, xs, sizeof(float) * (size_t)n);
        }
        if (st == REF_OK) {
            for (int64_t i = 0; i < n; i++) {
                if (e) e[o + i] = xs[i] - dec[i];
                if (dec_out) dec_out[o + i] = dec[i];
            }
        } else {
#pragma omp critical
            status = st;
        }
        free(xs); free(dec);
    }
    free(bs); free(bo);
    return status;
}

/* Decode a full payload (stage 1 or stage 2) into out (a10). */
int ref_qsgd_unpack(const ref_layer* layers, int32_t L, const int32_t* lbits, int32_t B,
                    const uint8_t* payload, float* out) {
    int64_t* bs = (int64_t*)malloc(sizeof(int64_t) * (L + 1));
    int64_t* bo = (int64_t*)malloc(sizeof(int64_t) * (L + 1));
    ref_layout(layers, L, lbits, B, bs, bo);
#pragma omp parallel for schedule(dynamic, 1)
    for (int l = 0; l < L; l++) {
        int64_t n = layers[l].numel, o = layers[l].offset;
        if (lbits[l] > 0) {
            int64_t nb = nbuckets(n, B);
            for (int64_t j = 0; j < nb; j++) {
                int32_t nv = (int32_t)((n - j * B) < B ? (n - j * B) : B);
                unpack_record(payload + bo[l] + j * rec_bytes_full(lbits[l], B), nv, lbits[l], B, out + o + j * B);
            }
        } else {
            memcpy(out + o, payload + bo[l], sizeof(float) * (size_t)n);
        }
    }
    free(bs); free(bo);
    return REF_OK;
}

/* Shard bounds over records (R13): r_0=0, r_W=R, r_j = min{r: off(r) >= floor(j*S/W)}. */
int ref_shard_bounds(const ref_layer* layers, int32_t L, const int32_t* lbits, int32_t B,
                     int32_t W, int64_t* rec_bounds /*W+1*/, int64_t* byte_bounds /*W+1*/) {
    int64_t* bs = (int64_t*)malloc(sizeof(int64_t) * (L + 1));
    int64_t* bo = (int64_t*)malloc(sizeof(int64_t) * (L + 1));
    int64_t S = ref_layout(layers, L, lbits, B, bs, bo);
    int64_t R = bs[L];
    for (int j = 0; j <= W; j++) {
        int64_t target = (int64_t)((__int128)j * S / W);
        /* linear scan over records: offset of record r */
        int64_t r = 0, off = 0;
        int found = 0;
        for (int l = 0; l < L && !found; l++) {
            int64_t nb = bs[l + 1] - bs[l];
            for (int64_t t = 0; t < nb; t++) {
                int64_t o = bo[l] + (lbits[l] > 0 ? t * rec_bytes_full(lbits[l], B) : t * 4 * (int64_t)B);
                if (o >= target) { r = bs[l] + t; off = o; found = 1; break; }
            }
        }
        if (!found) { r = R; off = S; }
        if (j == 0) { r = 0; off = 0; }
        if (j == W) { r = R; off = S; }
        rec_bounds[j] = r;
        byte_bounds[j] = off;
    }
    free(bs); free(bo);
    return REF_OK;
}

/* W-rank compressed all-reduce, simulated sequentially (a8-a10, R13-R15):
 * stage 1 pack per rank (EF updated); W==1 -> out = dec(stage 1);
 * else every record: decode the W stage-1 records, sum in rank order (fp32),
 * multiply by fl(1/W), requantise on stream 1 with rank field 0xFFFFFFFF,
 * out = dec(stage 2).  g, e: W*N (rank-major); pay1: W*S; pay2: S.        */
int ref_qsgd_allreduce(const ref_layer* layers, int32_t L, const int32_t* lbits, int32_t B,
                       uint64_t seed, uint64_t step, int32_t W, int64_t N, const float* g,
                       float* e, uint8_t* pay1, uint8_t* pay2, float* out) {
    int64_t* bs = (int64_t*)malloc(sizeof(int64_t) * (L + 1));
    int64_t* bo = (int64_t*)malloc(sizeof(int64_t) * (L + 1));
    int64_t S = ref_layout(layers, L, lbits, B, bs, bo);
    int st = REF_OK;
    for (int w = 0; w < W && st == REF_OK; w++)
        st = ref_qsgd_pack(layers, L, lbits, B, seed, (uint32_t)w, step, g + (int64_t)w * N,
                           e ? e + (int64_t)w * N : NULL, pay1 + (int64_t)w * S, NULL);
    if (st) { free(bs); free(bo); return st; }
    if (W == 1) {
        memcpy(pay2, pay1, (size_t)S);
        st = ref_qsgd_unpack(layers, L, lbits, B, pay2, out);
        free(bs); free(bo);
        return st;
    }
    float invW = 1.0f / (float)W;
    float* tmp = (float*)malloc(sizeof(float) * B);
    float* acc = (float*)malloc(sizeof(float) * B);
    float* dec2 = (float*)malloc(sizeof(float) * B);
    float* u = (float*)malloc(sizeof(float) * B);
    uint32_t* q = (uint32_t*)malloc(sizeof(uint32_t) * B);
    for (int l = 0; l < L && st == REF_OK; l++) {
        int64_t n = layers[l].numel, nb = bs[l + 1] - bs[l];
        for (int64_t j = 0; j < nb && st == REF_OK; j++) {
            int32_t nv = (int32_t)((n - j * B) < B ? (n - j * B) : B);
            for (int w = 0; w < W; w++) {
                const uint8_t* src = pay1 + (int64_t)w * S + bo[l];
                if (lbits[l] > 0) unpack_record(src + j * rec_bytes_full(lbits[l], B), nv, lbits[l], B, tmp);
                else memcpy(tmp, src + j * 4 * (int64_t)B, sizeof(float) * nv);
                for (int i = 0; i < nv; i++) acc[i] = (w == 0) ? tmp[i] : acc[i] + tmp[i];
            }
            for (int i = 0; i < nv; i++) acc[i] = acc[i] * invW;
            if (lbits[l] > 0) {
                float mn, unit;
                ref_bucket_uniforms(seed, 0xFFFFFFFFu, step, 1u, bs[l] + j, B, nv, u);
                st = ref_quantize_bucket(acc, nv, lbits[l], u, q, dec2, &mn, &unit);
                if (st == REF_OK)
                    pack_record(pay2 + bo[l] + j * rec_bytes_full(lbits[l], B), q, nv, lbits[l], B, mn, unit);
            } else {
                memcpy(pay2 + bo[l] + j * 4 * (int64_t)B, acc, sizeof(float) * nv);
            }
        }
    }
    if (st == REF_OK) st = ref_qsgd_unpack(layers, L, lbits, B, pay2, out);
    free(tmp); free(acc); free(dec2); free(u); free(q); free(bs); free(bo);
    return st;
}

/* Owner side of the exchange for one shard (R13): records [r0, r1) whose stage-1
 * bytes from the W ranks sit rank-major in recv (W x shard_bytes, shard starting at
 * byte0).  Writes the stage-2 records at their payload offsets in pay2. */
int ref_qsgd_reduce_shard(const ref_layer* layers, int32_t L, const int32_t* lbits, int32_t B, uint64_t seed,
                          uint64_t step, int32_t W, const uint8_t* recv, int64_t r0, int64_t r1, int64_t byte0,
                          int64_t shard_bytes, uint8_t* pay2) {
    int64_t* bs = (int64_t*)malloc(sizeof(int64_t) * (L + 1));
    int64_t* bo = (int64_t*)malloc(sizeof(int64_t) * (L + 1));
    ref_layout(layers, L, lbits, B, bs, bo);
    float invW = 1.0f / (float)W;
    float* tmp = (float*)malloc(sizeof(float) * B);
    float* acc = (float*)malloc(sizeof(float) * B);
    float* dec2 = (float*)malloc(sizeof(float) * B);
    float* u = (float*)malloc(sizeof(float) * B);
    uint32_t* q = (uint32_t*)malloc(sizeof(uint32_t) * B);
    int st = REF_OK;
    for (int l = 0; l < L && st == REF_OK; l++) {
        int64_t n = layers[l].numel;
        for (int64_t j = 0; j < bs[l + 1] - bs[l] && st == REF_OK; j++) {
            int64_t r = bs[l] + j;
            if (r < r0 || r >= r1) continue;
            int32_t nv = (int32_t)((n - j * B) < B ? (n - j * B) : B);
            int64_t roff = bo[l] + (lbits[l] > 0 ? j * rec_bytes_full(lbits[l], B) : j * 4 * (int64_t)B);
            for (int w = 0; w < W; w++) {
                const uint8_t* src = recv + (int64_t)w * shard_bytes + (roff - byte0);
                if (lbits[l] > 0) unpack_record(src, nv, lbits[l], B, tmp);
                else memcpy(tmp, src, sizeof(float) * nv);
                for (int i = 0; i < nv; i++) acc[i] = (w == 0) ? tmp[i] : acc[i] + tmp[i];
            }
            for (int i = 0; i < nv; i++) acc[i] = acc[i] * invW;
            if (lbits[l] > 0) {
                float mn, unit;
                ref_bucket_uniforms(seed, 0xFFFFFFFFu, step, 1u, r, B, nv, u);
                st = ref_quantize_bucket(acc, nv, lbits[l], u, q, dec2, &mn, &unit);
                if (st == REF_OK) pack_record(pay2 + roff, q, nv, lbits[l], B, mn, unit);
            } else {
                memcpy(pay2 + roff, acc, sizeof(float) * nv);
            }
        }
    }
    free(tmp); free(acc); free(dec2); free(u); free(q); free(bs); free(bo);
    return st;
}

/* ------------------------------------------------------------------------ */
/* TopK (R8-R10).                                                             */
/* ------------------------------------------------------------------------ */
int64_t ref_topk_k(int64_t n, int32_t ppm) {
    int64_t k = ((int64_t)ppm * n + 999999) / 1000000;
    if (k < 1) k = 1;
    if (k > n) k = n;
    return k;
}

typedef struct { uint32_t key; uint32_t idx; } kv_t;

static int cmp_key_desc_idx_asc(const void* a, const void* b) {
    const kv_t* x = (const kv_t*)a;
    const kv_t* y = (const kv_t*)b;
    if (x->key != y->key) return x->key > y->key ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx ? 1 : 0);
}
static int cmp_u32(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}
static uint32_t fkey(float v) { uint32_t u; memcpy(&u, &v, 4); return u & 0x7fffffffu; }

/* Indices (ascending) of the k largest |x|, ties to lower index. */
int ref_topk_select(const float* x, int64_t n, int64_t k, uint32_t* idx) {
    kv_t* a = (kv_t*)malloc(sizeof(kv_t) * (size_t)n);
    if (!a) return REF_ENOMEM;
    for (int64_t i = 0; i < n; i++) {
        if (!isfinite(x[i])) { free(a); return REF_ENONFINITE; }
        a[i].key = fkey(x[i]); a[i].idx = (uint32_t)i;
    }
    qsort(a, (size_t)n, sizeof(kv_t), cmp_key_desc_idx_asc);
    for (int64_t i = 0; i < k; i++) idx[i] = a[i].idx;
    qsort(idx, (size_t)k, sizeof(uint32_t), cmp_u32);
    free(a);
    return REF_OK;
}

static int cmp_dbl_asc(const void* a, const void* b) {
    double x = *(const double*)a, y = *(const double*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

/* TopK profile (a3): err = sqrt(sum of the n-k smallest squares), bits = 64k. */
int ref_topk_profile(const ref_layer* layers, int32_t L, const float* g, const float* e,
                     const int32_t* ppm, int32_t K, double* err, int64_t* bits) {
    for (int l = 0; l < L; l++) {
        int64_t n = layers[l].numel, o = layers[l].offset;
        if (!layers[l].compress) {
            for (int j = 0; j < K; j++) { err[l * K + j] = 0.0; bits[l * K + j] = 32 * n; }
            continue;
        }
        double* sq = (double*)malloc(sizeof(double) * (size_t)n);
        if (!sq) return REF_ENOMEM;
        for (int64_t i = 0; i < n; i++) {
            float x = canon_x(g[o + i], e ? e + o : NULL, i);
            if (!isfinite(x)) { free(sq); return REF_ENONFINITE; }
            sq[i] = (double)x * (double)x;
        }
        qsort(sq, (size_t)n, sizeof(double), cmp_dbl_asc);
        for (int j = 0; j < K; j++) {
            int64_t k = ref_topk_k(n, ppm[j]);
            double s = 0.0;
            for (int64_t i = 0; i < n - k; i++) s += sq[i];
            err[l * K + j] = sqrt(s);
            bits[l * K + j] = 64 * k;
        }
        free(sq);
    }
    return REF_OK;
}

/* TopK payload byte offsets: per layer 8*k (idx,val) pairs, lossless 4n, each layer
 * block 16-byte aligned (zero padding). */
int64_t ref_topk_layout(const ref_layer* layers, int32_t L, const int32_t* lppm, int64_t* byte_off) {
    int64_t off = 0;
    for (int l = 0; l < L; l++) {
        byte_off[l] = off;
        off += lppm[l] > 0 ? 8 * ref_topk_k(layers[l].numel, lppm[l]) : 4 * layers[l].numel;
        off = (off + 15) & ~(int64_t)15; /* 16-byte aligned layer blocks (R9) */
    }
    byte_off[L] = off;
    return off;
}

/* TopK compress of one rank (a8): payload pairs (u32 idx, f32 val) ascending idx;
 * e <- x with kept entries zeroed; lossless layers raw.  lppm[l]=0 -> lossless. */
int ref_topk_pack(const ref_layer* layers, int32_t L, const int32_t* lppm, const float* g,
                  float* e, uint8_t* payload) {
    int64_t* bo = (int64_t*)malloc(sizeof(int64_t) * (L + 1));
    ref_topk_layout(layers, L, lppm, bo);
    int st = REF_OK;
    for (int l = 0; l < L && st == REF_OK; l++) {
        int64_t n = layers[l].numel, o = layers[l].offset;
        float* xs = (float*)malloc(sizeof(float) * (size_t)n);
        for (int64_t i = 0; i < n; i++) xs[i] = canon_x(g[o + i], e ? e + o : NULL, i);
        if (lppm[l] > 0) {
            int64_t k = ref_topk_k(n, lppm[l]);
            uint32_t* idx = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)k);
            st = ref_topk_select(xs, n, k, idx);
            if (st == REF_OK) {
                for (int64_t t = 0; t < k; t++) {
                    memcpy(payload + bo[l] + 8 * t, &idx[t], 4);
                    memcpy(payload + bo[l] + 8 * t + 4, &xs[idx[t]], 4);
                }
                if (e) {
                    for (int64_t i = 0; i < n; i++) e[o + i] = xs[i];
                    for (int64_t t = 0; t < k; t++) e[o + idx[t]] = 0.0f;
                }
            }
            free(idx);
        } else {
            memcpy(payload + bo[l], xs, sizeof(float) * (size_t)n);
            if (e) for (int64_t i = 0; i < n; i++) e[o + i] = 0.0f;
        }
        free(xs);
    }
    free(bo);
    return st;
}

/* W-rank TopK exchange (a9-a10, R10): out = 0; for w in rank order, for each kept
 * (i,v): out[i] = out[i] + v*fl(1/W); lossless layers: out = (sum_w x_w)*fl(1/W). */
int ref_topk_allreduce(const ref_layer* layers, int32_t L, const int32_t* lppm, int32_t W,
                       int64_t N, const float* g, float* e, uint8_t* pays /*W*S*/, float* out) {
    int64_t* bo = (int64_t*)malloc(sizeof(int64_t) * (L + 1));
    int64_t S = ref_topk_layout(layers, L, lppm, bo);
    int st = REF_OK;
    for (int w = 0; w < W && st == REF_OK; w++)
        st = ref_topk_pack(layers, L, lppm, g + (int64_t)w * N, e ? e + (int64_t)w * N : NULL,
                           pays + (int64_t)w * S);
    float invW = 1.0f / (float)W;
    for (int l = 0; l < L && st == REF_OK; l++) {
        int64_t n = layers[l].numel, o = layers[l].offset;
        if (lppm[l] > 0) {
            int64_t k = ref_topk_k(n, lppm[l]);
            for (int64_t i = 0; i < n; i++) out[o + i] = 0.0f;
            for (int w = 0; w < W; w++)
                for (int64_t t = 0; t < k; t++) {
                    uint32_t idx; float v;
                    memcpy(&idx, pays + (int64_t)w * S + bo[l] + 8 * t, 4);
                    memcpy(&v, pays + (int64_t)w * S + bo[l] + 8 * t + 4, 4);
                    out[o + idx] = out[o + idx] + v * invW;
                }
        } else {
            for (int64_t i = 0; i < n; i++) {
                float s = 0.0f;
                for (int w = 0; w < W; w++) {
                    float v;
                    memcpy(&v, pays + (int64_t)w * S + bo[l] + 4 * i, 4);
                    s = (w == 0) ? v : s + v;
                }
                out[o + i] = s * invW;
            }
        }
    }
    free(bo);
    return st;
}

/* ------------------------------------------------------------------------ */
/* PowerSGD (R11, R12): fp64 power iteration, modified Gram-Schmidt.          */
/* Column-major factors: P[j*m+i] (m x r), Q[j*k+c] (k x r).                   */
/* ------------------------------------------------------------------------ */
/* Q0[j][c] = 2u-1, u from Philox ctr=((j*k+c)>>2, layer, step_lo32, 2), word (j*k+c)&3. */
void ref_psgd_init_q(uint64_t seed, uint32_t layer, uint64_t step, int32_t k, int32_t r, double* Q) {
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    for (int j = 0; j < r; j++)
        for (int c = 0; c < k; c++) {
            uint64_t t = (uint64_t)j * (uint64_t)k + (uint64_t)c;
            uint32_t ctr[4] = {(uint32_t)(t >> 2), layer, (uint32_t)step, 2u};
            uint32_t o[4];
            ref_philox4x32_10(ctr, key, o);
            float u = word_to_u(o[t & 3]);
            Q[(int64_t)j * k + c] = (double)(2.0f * u - 1.0f);
        }
}

/* P = M Q  (M row-major m x k, double) */
static void mat_mq(const double* M, int64_t m, int64_t k, int32_t r, const double* Q, double* P) {
    for (int j = 0; j < r; j++)
        for (int64_t i = 0; i < m; i++) {
            double s = 0.0;
            for (int64_t c = 0; c < k; c++) s += M[i * k + c] * Q[j * k + c];
            P[j * m + i] = s;
        }
}
/* Q = M^T P: Q[j][c] = sum over i = 0, 1, ..., m-1 (in that order) of M[i][c] P[j][i].
 * The loops run i outside c so M is read row by row; every Q[j][c] still accumulates its
 * terms in ascending i from 0.0, so the result is the plain dot product's, bit for bit. */
static void mat_mtp(const double* M, int64_t m, int64_t k, int32_t r, const double* P, double* Q) {
    for (int j = 0; j < r; j++) {
        double* q = Q + (int64_t)j * k;
        for (int64_t c = 0; c < k; c++) q[c] = 0.0;
        for (int64_t i = 0; i < m; i++) {
            const double pji = P[j * m + i];
            const double* row = M + i * k;
            for (int64_t c = 0; c < k; c++) q[c] += row[c] * pji;
        }
    }
}
/* Modified Gram-Schmidt with one reorthogonalisation sweep ("twice is enough") on
 * the columns of P (in place).  A column whose norm after the projections is <= 1e-12
 * of its norm before them is numerically dependent on the previous columns and is
 * set to 0 (R11: "a column with norm 0 stays 0", read in floating point).  A single
 * MGS sweep loses orthogonality on nearly dependent columns (tests/test_oracle_psgd.py
 * rank-deficient pin); the second sweep restores it to round-off. */
void ref_mgs(double* P, int64_t m, int32_t r) {
    for (int j = 0; j < r; j++) {
        double* pj = P + (int64_t)j * m;
        double n0 = 0.0;
        for (int64_t t = 0; t < m; t++) n0 += pj[t] * pj[t];
        n0 = sqrt(n0);
        for (int sweep = 0; sweep < 2; sweep++)
            for (int i = 0; i < j; i++) {
                const double* pi = P + (int64_t)i * m;
                double d = 0.0;
                for (int64_t t = 0; t < m; t++) d += pi[t] * pj[t];
                for (int64_t t = 0; t < m; t++) pj[t] -= d * pi[t];
            }
        double nrm = 0.0;
        for (int64_t t = 0; t < m; t++) nrm += pj[t] * pj[t];
        nrm = sqrt(nrm);
        int zero = !(nrm > 1e-12 * n0);
        for (int64_t t = 0; t < m; t++) pj[t] = zero ? 0.0 : pj[t] / nrm;
    }
}

/* `steps` power steps from Q (in/out): P = MQ; P <- MGS(P); Q = M^T P. */
void ref_psgd_power(const double* M, int64_t m, int64_t k, int32_t r, int32_t steps, double* P, double* Q) {
    for (int s = 0; s < steps; s++) {
        mat_mq(M, m, k, r, Q, P);
        ref_mgs(P, m, r);
        mat_mtp(M, m, k, r, P, Q);
    }
}

/* ||M - P Q^T||_F computed directly (fp64). */
double ref_psgd_err(const double* M, int64_t m, int64_t k, int32_t r, const double* P, const double* Q) {
    double s = 0.0;
    for (int64_t i = 0; i < m; i++)
        for (int64_t c = 0; c < k; c++) {
            double a = 0.0;
            for (int j = 0; j < r; j++) a += P[(int64_t)j * m + i] * Q[(int64_t)j * k + c];
            double d = M[i * k + c] - a;
            s += d * d;
        }
    return sqrt(s);
}

static int psgd_lossless(int64_t m, int64_t k, int32_t r) { return (int64_t)r * (m + k) >= m * k; }

/* PowerSGD profile (a4): for each candidate rank separately (literal, no prefix
 * sharing): Q0 from stream 2, `steps` power steps, err = ||M - P Q^T||_F.    */
int ref_psgd_profile(const ref_layer* layers, int32_t L, const float* g, const float* e,
                     const int32_t* ranks, int32_t K, int32_t steps, uint64_t seed, uint64_t step,
                     double* err, int64_t* bits) {
    for (int l = 0; l < L; l++) {
        int64_t n = layers[l].numel, o = layers[l].offset;
        if (!layers[l].compress || layers[l].rows <= 0) {
            for (int j = 0; j < K; j++) { err[l * K + j] = 0.0; bits[l * K + j] = 32 * n; }
            continue;
        }
        int64_t m = layers[l].rows, k = layers[l].cols;
        double* M = (double*)malloc(sizeof(double) * (size_t)n);
        for (int64_t i = 0; i < n; i++) {
            float x = canon_x(g[o + i], e ? e + o : NULL, i);
            if (!isfinite(x)) { free(M); return REF_ENONFINITE; }
            M[i] = (double)x;
        }
        for (int j = 0; j < K; j++) {
            int32_t r = ranks[j];
            if (psgd_lossless(m, k, r)) { err[l * K + j] = 0.0; bits[l * K + j] = 32 * n; continue; }
            double* P = (double*)malloc(sizeof(double) * (size_t)(m * r));
            double* Q = (double*)malloc(sizeof(double) * (size_t)(k * r));
            ref_psgd_init_q(seed, (uint32_t)l, step, (int32_t)k, r, Q);
            ref_psgd_power(M, m, k, r, steps, P, Q);
            err[l * K + j] = ref_psgd_err(M, m, k, r, P, Q);
            bits[l * K + j] = 32 * (int64_t)r * (m + k);
            free(P); free(Q);
        }
        free(M);
    }
    return REF_OK;
}

/* PowerSGD compressed all-reduce over W simulated ranks, one warm-started step
 * (a8-a10, PowerSGD as used via torch hooks):
 *   P_w = M_w Q; Pbar = (sum_w P_w)/W; Phat = MGS(Pbar); Q_w = M_w^T Phat;
 *   Qbar = (sum_w Q_w)/W; out = Phat Qbar^T; e_w <- x_w - out; Q <- Qbar.
 * lrank[l] = 0 or a lossless-equivalent rank -> layer exchanged raw (mean).
 * Qstate: per layer k x lrank doubles at qoff[l] (caller initialises).      */
int ref_psgd_allreduce(const ref_layer* layers, int32_t L, const int32_t* lrank, int32_t W,
                       int64_t N, const float* g, float* e, double* Qstate, const int64_t* qoff,
                       float* out, double* Pout /*nullable: per layer m x r at poff*/,
                       const int64_t* poff) {
    float invW = 1.0f / (float)W;
    for (int l = 0; l < L; l++) {
        int64_t n = layers[l].numel, o = layers[l].offset;
        int32_t r = lrank[l];
        int64_t m = layers[l].rows, k = layers[l].cols;
        int lossless = (r <= 0) || !layers[l].compress || m <= 0 || psgd_lossless(m, k, r);
        float* xs = (float*)malloc(sizeof(float) * (size_t)(n * W));
        for (int w = 0; w < W; w++)
            for (int64_t i = 0; i < n; i++)
                xs[w * n + i] = canon_x(g[w * N + o + i], e ? e + w * N + o : NULL, i);
        if (lossless) {
            for (int64_t i = 0; i < n; i++) {
                float s = 0.0f;
                for (int w = 0; w < W; w++) s = (w == 0) ? xs[w * n + i] : s + xs[w * n + i];
                out[o + i] = s * invW;
            }
            if (e) for (int w = 0; w < W; w++) for (int64_t i = 0; i < n; i++) e[w * N + o + i] = 0.0f;
            free(xs);
            continue;
        }
        double* Q = Qstate + qoff[l];
        double* M = (double*)malloc(sizeof(double) * (size_t)n);
        double* Pw = (double*)malloc(sizeof(double) * (size_t)(m * r));
        double* Pb = (double*)calloc((size_t)(m * r), sizeof(double));
        double* Qw = (double*)malloc(sizeof(double) * (size_t)(k * r));
        double* Qb = (double*)calloc((size_t)(k * r), sizeof(double));
        for (int w = 0; w < W; w++) {
            for (int64_t i = 0; i < n; i++) M[i] = (double)xs[w * n + i];
            mat_mq(M, m, k, r, Q, Pw);
            for (int64_t t = 0; t < m * r; t++) Pb[t] += Pw[t];
        }
        for (int64_t t = 0; t < m * r; t++) Pb[t] /= (double)W;
        ref_mgs(Pb, m, r);
        for (int w = 0; w < W; w++) {
            for (int64_t i = 0; i < n; i++) M[i] = (double)xs[w * n + i];
            mat_mtp(M, m, k, r, Pb, Qw);
            for (int64_t t = 0; t < k * r; t++) Qb[t] += Qw[t];
        }
        for (int64_t t = 0; t < k * r; t++) Qb[t] /= (double)W;
        for (int64_t i = 0; i < m; i++)
            for (int64_t c = 0; c < k; c++) {
                double a = 0.0;
                for (int j = 0; j < r; j++) a += Pb[(int64_t)j * m + i] * Qb[(int64_t)j * k + c];
                float af = (float)a;
                out[o + i * k + c] = af;
                if (e) for (int w = 0; w < W; w++) e[w * N + o + i * k + c] = xs[w * n + i * k + c] - af;
            }
        memcpy(Q, Qb, sizeof(double) * (size_t)(k * r));
        if (Pout) memcpy(Pout + poff[l], Pb, sizeof(double) * (size_t)(m * r));
        free(M); free(Pw); free(Pb); free(Qw); free(Qb); free(xs);
    }
    return REF_OK;
}

/* ------------------------------------------------------------------------ */
/* Algorithm 1 DP with readings R16-R20.                   */
/* ------------------------------------------------------------------------ */
#define REF_METRIC_SQ 1u
#define REF_DISC_FLOOR 2u

int ref_solve(const double* err, const int64_t* bits, int32_t L, int32_t K, const int32_t* default_idx,
              const int32_t* compress, int32_t D, uint32_t flags, int32_t* choice, ref_solve_info* info) {
    if (L < 0 || K <= 0 || K > 255 || D <= 0) return REF_EINVAL;
    int32_t La = 0;
    for (int l = 0; l < L; l++) {
        int act = compress ? compress[l] : 1;
        choice[l] = -1;
        if (!act) continue;
        if (default_idx[l] < 0 || default_idx[l] >= K) return REF_EINVAL;
        for (int j = 0; j < K; j++) {
            if (!isfinite(err[l * K + j]) || err[l * K + j] < 0.0) return REF_ENONFINITE;
            if (bits[l * K + j] < 0) return REF_EINVAL;
        }
        La++;
    }
    memset(info, 0, sizeof(*info));
    info->n_active = La;
    if (La == 0) return REF_OK;
    int32_t* act = (int32_t*)malloc(sizeof(int32_t) * La);
    for (int l = 0, a = 0; l < L; l++) if (!compress || compress[l]) act[a++] = l;
    double* me = (double*)malloc(sizeof(double) * (size_t)La * K);
    for (int a = 0; a < La; a++)
        for (int j = 0; j < K; j++) {
            double v = err[act[a] * K + j];
            me[a * K + j] = (flags & REF_METRIC_SQ) ? v * v : v;
        }
    /* Alg.1 line 2: Emax = error of the default parameters (layer order, fp64) */
    double emax = 0.0;
    int64_t defbits = 0;
    for (int a = 0; a < La; a++) {
        emax += me[a * K + default_idx[act[a]]];
        defbits += bits[act[a] * K + default_idx[act[a]]];
    }
    /* Alg.1 lines 3-5: discretise, step Emax/D (R16: ceil; R17: infeasible if > D) */
    int32_t* disc = (int32_t*)malloc(sizeof(int32_t) * (size_t)La * K);
    for (int a = 0; a < La; a++)
        for (int j = 0; j < K; j++) {
            double v = me[a * K + j];
            int32_t d;
            if (emax == 0.0) {
                d = (v == 0.0) ? 0 : -1;
            } else {
                double q = (v * (double)D) / emax;
                double r = (flags & REF_DISC_FLOOR) ? floor(q) : ceil(q);
                d = (r > (double)D) ? -1 : (int32_t)r;
            }
            disc[a * K + j] = d;
        }
    /* Alg.1 lines 6-22 with the min-update init (R18) and strict < (R19) */
    const int64_t INF = INT64_MAX;
    int64_t* prev = (int64_t*)malloc(sizeof(int64_t) * (size_t)(D + 1));
    int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)(D + 1));
    uint8_t* PD = (uint8_t*)malloc((size_t)La * (D + 1));
    for (int e = 0; e <= D; e++) prev[e] = INF;
    prev[0] = 0;
    for (int a = 0; a < La; a++) {
        for (int e = 0; e <= D; e++) { cur[e] = INF; PD[(size_t)a * (D + 1) + e] = 0; }
        for (int c = 0; c < K; c++) {
            int32_t d = disc[a * K + c];
            if (d < 0) continue;
            for (int e = d; e <= D; e++) {
                if (prev[e - d] == INF) continue;
                int64_t t = prev[e - d] + bits[act[a] * K + c];
                if (t < cur[e]) { cur[e] = t; PD[(size_t)a * (D + 1) + e] = (uint8_t)c; }
            }
        }
        int64_t* sw = prev; prev = cur; cur = sw;
    }
    /* Alg.1 line 23: argmin, smallest e on ties (R19) */
    int64_t best = INF;
    int ebest = -1;
    for (int e = 0; e <= D; e++) if (prev[e] < best) { best = prev[e]; ebest = e; }
    int used_default = 0;
    if (ebest < 0) {
        used_default = 1;
    } else {
        /* lines 24-27: backtrack */
        int e = ebest;
        for (int a = La - 1; a >= 0; a--) {
            int c = PD[(size_t)a * (D + 1) + e];
            choice[act[a]] = c;
            e -= disc[a * K + c];
        }
        /* R20: never worse than the defaults, never above Emax in raw error */
        int64_t pb = 0;
        double pe = 0.0;
        for (int a = 0; a < La; a++) {
            pb += bits[act[a] * K + choice[act[a]]];
            pe += me[a * K + choice[act[a]]];
        }
        if (pb > defbits || pe > emax) used_default = 1;
    }
    if (used_default)
        for (int a = 0; a < La; a++) choice[act[a]] = default_idx[act[a]];
    int64_t tb = 0;
    double te = 0.0;
    for (int a = 0; a < La; a++) {
        tb += bits[act[a] * K + choice[act[a]]];
        te += me[a * K + choice[act[a]]];
    }
    info->emax = emax;
    info->total_err = te;
    info->total_bits = tb;
    info->default_bits = defbits;
    info->used_default = used_default;
    free(act); free(me); free(disc); free(prev); free(cur); free(PD);
    return REF_OK;
}
