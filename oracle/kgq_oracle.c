/*
 * kgq_oracle.c -- CPU restatement of the reference quantizer / SpMM / ReLU-mask
 * path.  TEST INFRASTRUCTURE ONLY: this file is the parity checker for the
 * sm_100a kernels in paper_2212_04540_b200/csrc.  It is linked by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg,
 * never by the product path.
 *
 * Every function restates the reference (kgact, /root/reference/pkg/src/kgact)
 * and cites the lines it follows.  Floating point is plain IEEE fp32 with
 * -ffp-contract=off (no FMA contraction), which is what numpy's elementwise
 * float32 loops compute.
 *
 * Parity is pinned by tests/golden/ (npz), generated from the reference itself
 * by tests/golden/make_golden.py (see tests/test_oracle.py).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define KGQ_MODE_NEAREST 0      /* np.rint, quantize.py:129-130            */
#define KGQ_MODE_SR_FAST 1      /* Philox4x32-7, 16-bit uniforms (ours)    */
#define KGQ_MODE_SR_COMPAT 2    /* numpy Philox4x64-10 stream, quantize.py:61-102 */
#define KGQ_MODE_SR_NOISE 3     /* caller-supplied float64 uniforms        */

/* ------------------------------------------------------------------ */
/* Philox4x64-10 exactly as numpy's Philox bit generator (the reference's
 * RandomStream uses Generator(Philox(key=[seed, tid])), quantize.py:80-81,95).
 * numpy pre-increments the 256-bit counter before each block, so the first
 * block of a fresh generator is counter (1,0,0,0).                        */
static inline void mulhilo64(uint64_t a, uint64_t b, uint64_t *hi, uint64_t *lo) {
    __uint128_t p = (__uint128_t)a * (__uint128_t)b;
    *lo = (uint64_t)p;
    *hi = (uint64_t)(p >> 64);
}

void oracle_philox4x64_10(const uint64_t ctr_in[4], const uint64_t key_in[2], uint64_t out[4]) {
    uint64_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint64_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; r++) {
        if (r) { k0 += 0x9E3779B97F4A7C15ULL; k1 += 0xBB67AE8584CAA73BULL; }
        uint64_t hi0, lo0, hi1, lo1;
        mulhilo64(0xD2E7470EE14C6C93ULL, c0, &hi0, &lo0);
        mulhilo64(0xCA5A826395121157ULL, c2, &hi1, &lo1);
        uint64_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Philox4x32-R (Random123 constants).  R = 10 is the Random123 reference
 * (pinned by its KAT); our "fast" SR mode uses R = 7.          */
#define ORACLE_FAST_ROUNDS 7
void oracle_philox4x32_r(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4], int rounds) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < rounds; r++) {
        if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0, n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1, n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    oracle_philox4x32_r(ctr_in, key_in, out, 10);
}

/* Compat stream: element k of quantization group g (group = row of the
 * (-1, G) view) draws word k%4 of numpy block g*ceil(G/4) + k/4 (counter is
 * that +1), uniform = (raw >> 11) * 2^-53.  quantize.py:83-96.            */
uint64_t oracle_compat_raw53(uint64_t seed, uint64_t tid, uint64_t g, int64_t G, int64_t k) {
    uint64_t bpr = (uint64_t)((G + 3) / 4);
    uint64_t ctr[4] = {g * bpr + (uint64_t)(k / 4) + 1u, 0, 0, 0};
    uint64_t key[2] = {seed, tid};
    uint64_t out[4];
    oracle_philox4x64_10(ctr, key, out);
    return out[k & 3] >> 11;
}

/* Fast stream (our design): key = (lo32 seed,
 * hi32 seed ^ hi32 tid), counter = (call, lo32 g, hi32 g, lo32 tid).  Element
 * k of group g: call = 4*(k>>5) + ((k>>2)&3), word k&3, half (k>>4)&1 (low
 * half first).  Uniform = u16 / 65536.                                     */
uint32_t oracle_fast_u16(uint64_t seed, uint64_t tid, uint64_t g, int64_t k) {
    uint32_t call = (uint32_t)(4 * (k >> 5) + ((k >> 2) & 3));
    uint32_t ctr[4] = {call, (uint32_t)g, (uint32_t)(g >> 32), (uint32_t)tid};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32) ^ (uint32_t)(tid >> 32)};
    uint32_t out[4];
    oracle_philox4x32_r(ctr, key, out, ORACLE_FAST_ROUNDS);
    return (out[k & 3] >> (16 * ((k >> 4) & 1))) & 0xFFFFu;
}

/* All G draws of group g at once: each Philox call yields 8 of them (4 words
 * x 2 halves), the same values oracle_fast_u16 gives element by element. */
static void fast_group_u16(uint64_t seed, uint64_t tid, uint64_t g, int64_t G, uint16_t *buf) {
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32) ^ (uint32_t)(tid >> 32)};
    int64_t n_calls = 4 * ((G + 31) / 32);
    for (int64_t c = 0; c < n_calls; c++) {
        uint32_t ctr[4] = {(uint32_t)c, (uint32_t)g, (uint32_t)(g >> 32), (uint32_t)tid};
        uint32_t out[4];
        oracle_philox4x32_r(ctr, key, out, ORACLE_FAST_ROUNDS);
        for (int h = 0; h < 2; h++)
            for (int w = 0; w < 4; w++) {
                int64_t k = 32 * (c >> 2) + 16 * h + 4 * (c & 3) + w;
                if (k < G) buf[k] = (uint16_t)((out[w] >> (16 * h)) & 0xFFFFu);
            }
    }
}

void oracle_fast_noise_u16(uint64_t seed, uint64_t tid, int64_t n_groups, int64_t G, uint16_t *out) {
    for (int64_t g = 0; g < n_groups; g++)
        for (int64_t k = 0; k < G; k++)
            out[g * G + k] = (uint16_t)oracle_fast_u16(seed, tid, (uint64_t)g, k);
}

void oracle_compat_noise_raw53(uint64_t seed, uint64_t tid, int64_t n_groups, int64_t G, uint64_t *out) {
    uint64_t bpr = (uint64_t)((G + 3) / 4);
    uint64_t key[2] = {seed, tid};
    for (int64_t g = 0; g < n_groups; g++)
        for (int64_t b = 0; b < (int64_t)bpr; b++) {
            uint64_t ctr[4] = {(uint64_t)g * bpr + (uint64_t)b + 1u, 0, 0, 0};
            uint64_t o[4];
            oracle_philox4x64_10(ctr, key, o);
            for (int w = 0; w < 4 && 4 * b + w < G; w++) out[g * G + 4 * b + w] = o[w] >> 11;
        }
}

/* ------------------------------------------------------------------ */
/* quantize_tensor, quantize.py:177-196 (with _scale_rows :116-125,
 * _round_block :128-132, pack_codes :213-233) over the (-1, G) view.     */
static inline float f32_div(float a, float b) { volatile float q = a / b; return q; }

static void quantize_groups(const float *x, int64_t g0, int64_t g1, int64_t G, int bits, int mode,
                            uint64_t seed, uint64_t tid, int64_t goff, const double *noise,
                            uint8_t *codes, float *ranges, float *offsets, uint8_t *scratch,
                            uint16_t *noise16) {
    const int64_t gbytes = (G * bits + 7) / 8;
    const float B = (float)((1u << bits) - 1u);
    const uint64_t bpr = (uint64_t)((G + 3) / 4);
    for (int64_t g = g0; g < g1; g++) {
        const float *row = x + g * G;
        float mn = row[0], mx = row[0];
        for (int64_t k = 1; k < G && mn == mn; k++) { /* x.min / x.max, :184-185 */
            if (row[k] != row[k]) { mn = mx = row[k]; break; }   /* numpy propagates NaN */
            if (row[k] < mn) mn = row[k];
            if (row[k] > mx) mx = row[k];
        }
        float r = mx - mn;                           /* fp32 range, :185        */
        float z = mn;
        ranges[g] = r;
        offsets[g] = z;
        uint64_t blk_cache = ~0ULL;
        uint64_t words64[4] = {0, 0, 0, 0};
        for (int64_t k = 0; k < G; k++) {
            float s;
            if (r > 0.0f) {                           /* _scale_rows :120-122    */
                float a = row[k] - z;
                s = f32_div(a, r);
                s = s * B;
            } else {
                s = 0.0f;                             /* scaled[r == 0] = 0 :123 */
            }
            if (s < 0.0f) s = 0.0f;                   /* clip :125               */
            if (s > B) s = B;
            if (s != s) s = 0.0f;                     /* inf/inf: numpy's NaN cast gives code 0 */
            float code;
            if (mode == KGQ_MODE_NEAREST) {
                code = rintf(s);                      /* np.rint, half-even :130 */
            } else {
                float fl = floorf(s);
                float frac = s - fl;
                double u;
                if (mode == KGQ_MODE_SR_FAST) {
                    if (k == 0) fast_group_u16(seed, tid, (uint64_t)(g + goff), G, noise16);
                    u = (double)noise16[k] * (1.0 / 65536.0);
                } else if (mode == KGQ_MODE_SR_COMPAT) {
                    uint64_t blk = (uint64_t)(g + goff) * bpr + (uint64_t)(k / 4) + 1u;
                    if (blk != blk_cache) {
                        uint64_t ctr[4] = {blk, 0, 0, 0};
                        uint64_t key[2] = {seed, tid};
                        oracle_philox4x64_10(ctr, key, words64);
                        blk_cache = blk;
                    }
                    u = (double)(words64[k & 3] >> 11) * (1.0 / 9007199254740992.0);
                } else {
                    u = noise[g * G + k];
                }
                code = fl + ((u < (double)frac) ? 1.0f : 0.0f);   /* :131-132 */
            }
            scratch[k] = (uint8_t)code;
        }
        uint8_t *dst = codes + g * gbytes;            /* pack LSB-first :213-233 */
        memset(dst, 0, (size_t)gbytes);
        for (int64_t k = 0; k < G; k++) {
            int64_t bit = k * bits;
            dst[bit >> 3] |= (uint8_t)(scratch[k] << (bit & 7));
        }
    }
}

typedef struct {
    const float *x; int64_t g0, g1, G; int bits, mode; uint64_t seed, tid; int64_t goff; const double *noise;
    uint8_t *codes; float *ranges, *offsets;
} qjob_t;

static void *quantize_worker(void *p) {
    qjob_t *j = (qjob_t *)p;
    uint8_t *scratch = (uint8_t *)malloc((size_t)j->G);
    uint16_t *noise16 = (uint16_t *)malloc((size_t)j->G * sizeof(uint16_t));
    quantize_groups(j->x, j->g0, j->g1, j->G, j->bits, j->mode, j->seed, j->tid, j->goff, j->noise,
                    j->codes, j->ranges, j->offsets, scratch, noise16);
    free(noise16);
    free(scratch);
    return NULL;
}

int oracle_quantize(const float *x, int64_t n_groups, int64_t G, int bits, int mode,
                    uint64_t seed, uint64_t tid, int64_t group_offset, const double *noise,
                    uint8_t *codes, float *ranges, float *offsets, int n_threads) {
    if (!(bits == 1 || bits == 2 || bits == 4 || bits == 8)) return 2;
    if (G < 1 || n_groups < 0) return 1;
    if (mode == KGQ_MODE_SR_NOISE && !noise) return 1;
    if (n_threads < 1) n_threads = 1;
    if (n_threads > 256) n_threads = 256;
    if (n_threads == 1 || n_groups < 2 * n_threads) {
        qjob_t j = {x, 0, n_groups, G, bits, mode, seed, tid, group_offset, noise, codes, ranges, offsets};
        quantize_worker(&j);
        return 0;
    }
    pthread_t th[256];
    qjob_t jobs[256];
    for (int t = 0; t < n_threads; t++) {
        int64_t g0 = n_groups * t / n_threads, g1 = n_groups * (t + 1) / n_threads;
        jobs[t] = (qjob_t){x, g0, g1, G, bits, mode, seed, tid, group_offset, noise, codes, ranges, offsets};
        pthread_create(&th[t], NULL, quantize_worker, &jobs[t]);
    }
    for (int t = 0; t < n_threads; t++) pthread_join(th[t], NULL);
    return 0;
}

/* dequantize_tensor, quantize.py:199-210 (+ unpack_codes :236-247):
 * out = (R * c) / B + Z in fp32, rows with R == 0 give exactly Z.         */
typedef struct {
    const uint8_t *codes; const float *ranges, *offsets; int64_t g0, g1, G; int bits; float *out;
} djob_t;

static void *dequantize_worker(void *p) {
    djob_t *j = (djob_t *)p;
    const int64_t gbytes = (j->G * j->bits + 7) / 8;
    const float B = (float)((1u << j->bits) - 1u);
    const unsigned mask = (1u << j->bits) - 1u;
    for (int64_t g = j->g0; g < j->g1; g++) {
        const uint8_t *src = j->codes + g * gbytes;
        float r = j->ranges[g], z = j->offsets[g];
        float *o = j->out + g * j->G;
        for (int64_t k = 0; k < j->G; k++) {
            int64_t bit = k * j->bits;
            unsigned c = (src[bit >> 3] >> (bit & 7)) & mask;
            if (r == 0.0f) { o[k] = z; continue; }
            float t = r * (float)c;
            t = f32_div(t, B);
            o[k] = t + z;
        }
    }
    return NULL;
}

int oracle_dequantize(const uint8_t *codes, const float *ranges, const float *offsets,
                      int64_t n_groups, int64_t G, int bits, float *out, int n_threads) {
    if (!(bits == 1 || bits == 2 || bits == 4 || bits == 8)) return 2;
    if (n_threads < 1) n_threads = 1;
    if (n_threads > 256) n_threads = 256;
    if (n_threads == 1 || n_groups < 2 * n_threads) {
        djob_t j = {codes, ranges, offsets, 0, n_groups, G, bits, out};
        dequantize_worker(&j);
        return 0;
    }
    pthread_t th[256];
    djob_t jobs[256];
    for (int t = 0; t < n_threads; t++) {
        int64_t g0 = n_groups * t / n_threads, g1 = n_groups * (t + 1) / n_threads;
        jobs[t] = (djob_t){codes, ranges, offsets, g0, g1, G, bits, out};
        pthread_create(&th[t], NULL, dequantize_worker, &jobs[t]);
    }
    for (int t = 0; t < n_threads; t++) pthread_join(th[t], NULL);
    return 0;
}

/* spmm, tensorops.py:37-43 via scipy csr_matvecs: each output element is an
 * ascending-column fp32 accumulation acc = acc + a*x, no FMA (pinned by the
 * reference's own ordered oracle, test_tensorops.py:9-14, :64-71).        */
void oracle_spmm_csr(const int32_t *indptr, const int32_t *indices, const float *vals,
                     int64_t n_rows, const float *X, int64_t d, float *out) {
    for (int64_t i = 0; i < n_rows; i++) {
        float *o = out + i * d;
        for (int64_t k = 0; k < d; k++) o[k] = 0.0f;
        for (int32_t jj = indptr[i]; jj < indptr[i + 1]; jj++) {
            float a = vals[jj];
            const float *xr = X + (int64_t)indices[jj] * d;
            for (int64_t k = 0; k < d; k++) {
                volatile float p = a * xr[k];
                o[k] = o[k] + p;
            }
        }
    }
}

/* relu + BitMask.from_bool, tensorops.py:57-92: out = max(x, 0), mask bit
 * = x > 0, packed LSB-first over the flat element order.                  */
void oracle_relu_mask(const float *x, int64_t n, float *out, uint8_t *mask) {
    memset(mask, 0, (size_t)((n + 7) / 8));
    for (int64_t i = 0; i < n; i++) {
        float v = x[i];
        out[i] = !(v <= 0.0f) ? v : 0.0f;   /* np.maximum: NaN propagates */
        if (v > 0.0f) mask[i >> 3] |= (uint8_t)(1u << (i & 7));
    }
}
