/*
 * oracle/tlc_oracle.c -- plain, slow, obviously-correct CPU oracle of 3LC's
 * state-change compression pipeline (arXiv 1802.07389, Sec. 3).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load, call or link the
 * library built from this file.  The product path (paper_1802_07389_b200/)
 * never does, and this file shares no code, header, table or constant
 * generator with paper_1802_07389_b200/csrc/.
 *
 * Citations: "P:n" = PAPER.md line n, "S:n" = SPEC.md line n (the paper's
 * section/equation is named beside each).  "R<k>" = reading k of the paper
 * listed in DESIGN.md section 3, taken where the paper is silent/ambiguous.
 *
 * Arithmetic: fp32, as the paper (its state changes are 32-bit floats,
 * P:87-91).  Built with -O2 -ffp-contract=off -fno-fast-math on x86-64 (SSE,
 * FLT_EVAL_METHOD == 0), so each + - * / below is exactly one IEEE-754
 * round-to-nearest-even fp32 operation.
 *
 * Every step runs over the whole tensor before the next starts, in the order
 * the paper lists them; no fusion, no blocking.
 *
 * The element-wise loops carry "#pragma omp parallel for".  The default build
 * (no -fopenmp) ignores them; oracle.build(omp=True) compiles the same source
 * with -fopenmp for bench.py's cpu_baseline on all host cores.  Results are
 * identical: every element's operations are independent, and the one reduction
 * (the max of Eq. 1) is exact and order-free.  The zero-run coder (Sec. 3.3)
 * stays serial in both builds.
 *
 * Pinning (see tests/test_oracle_pins.py): every function is pinned by values
 * the paper or SPEC prints, closed forms, invariants or brute force.  The only
 * unpinned quantities are the paper's Table 2 s-rows (need real ResNet-110
 * gradients) -- "parity unpinned" for those, and they are not computed here.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Status values of this oracle (R6). */
enum {
    O_OK = 0,
    O_ERR_ARG = 1,       /* s outside [1,2), n == 0, short buffer  */
    O_ERR_NONFINITE = 2, /* NaN/Inf in u = buffer + T_in (R6)  */
    O_ERR_RANGE = 3,     /* max|u| * s overflows to Inf (R6)               */
    O_ERR_FORMAT = 4     /* malformed payload               */
};

/* ------------------------------------------------------------------------- */
/* Sec. 3.1, Fig. "fig:compression" step (1):                      */
/* "accumulates the input tensor into a local buffer": u = buffer + T_in.      */
void tlc_o_accumulate(const float *t, const float *buf, uint64_t n, float *u)
{
#pragma omp parallel for
    for (uint64_t i = 0; i < n; i++)
        u[i] = buf[i] + t[i];
}

/* Eq. 1: M = max(|T_in|) * s, taken over the accumulated sum u      */
/* (Fig. step 2 quantizes "the sum"; R2).  1 <= s < 2. */
/* Returns O_ERR_NONFINITE if some u is NaN/Inf, O_ERR_RANGE if M is Inf.    */
int tlc_o_scale(const float *u, uint64_t n, float s, float *M_out, float *maxabs_out)
{
    float a = 0.0f;
    int bad = 0;
    /* max is exact and order-free, so the -fopenmp build's reduction gives the same a */
#pragma omp parallel for reduction(max : a) reduction(| : bad)
    for (uint64_t i = 0; i < n; i++) {
        if (isnan(u[i]) || isinf(u[i]))
            bad = 1;
        else if (fabsf(u[i]) > a)
            a = fabsf(u[i]);
    }
    if (bad)
        return O_ERR_NONFINITE;
    float M = a * s;
    if (isinf(M))
        return O_ERR_RANGE;
    *maxabs_out = a;
    *M_out = M;
    return O_OK;
}

/* Eq. 2: T_quantized = round(T_in / M).                              */
/* round() = round half away from zero (R1): C99 roundf.  M == 0 only   */
/* when every u is zero; then every value is 0 (R5).                   */
void tlc_o_quantize(const float *u, uint64_t n, float M, int8_t *q)
{
#pragma omp parallel for
    for (uint64_t i = 0; i < n; i++) {
        if (M == 0.0f)
            q[i] = 0;
        else
            q[i] = (int8_t)roundf(u[i] / M);
    }
}

/* Eq. 3: T_out = M * T_quantized.                                    */
void tlc_o_dequantize(const int8_t *q, uint64_t n, float M, float *out)
{
#pragma omp parallel for
    for (uint64_t i = 0; i < n; i++)
        out[i] = M * (float)q[i];
}

/* Fig. step (a) "dequantizes the quantized data locally" and step (b)        */
/* "calculates remaining quantization errors and stores them in the local     */
/* buffer": buffer = u - M * q  (R7, R8).                         */
void tlc_o_residual(const float *u, const int8_t *q, uint64_t n, float M, float *buf)
{
#pragma omp parallel for
    for (uint64_t i = 0; i < n; i++)
        buf[i] = u[i] - M * (float)q[i];
}

/* ------------------------------------------------------------------------- */
/* Sec. 3.2 quartic encoding.  Output length: the padded length divided by 5. */
uint64_t tlc_o_quartic_len(uint64_t n)
{
    uint64_t L = n;
    while (L % 5 != 0)      /* step 4: "Pad it with zeros to make its length a multiple of 5" */
        L++;
    return L / 5;
}

/* Encoding steps 1-6, one pass per step.                         */
void tlc_o_quartic_encode(const int8_t *q, uint64_t n, uint8_t *out)
{
    uint64_t P = tlc_o_quartic_len(n);
    uint64_t L = 5 * P;
    uint8_t *a = (uint8_t *)malloc(L ? L : 1);
    /* step 1 "Element-wise add 1", step 2 "Type cast it to an unsigned 8-bit integer array" */
#pragma omp parallel for
    for (uint64_t i = 0; i < n; i++)
        a[i] = (uint8_t)(q[i] + 1);
    /* step 3 "Flatten it into a 1-D array": q is already flat (row-major).   */
    /* step 4 "Pad it with zeros" -- the pad is digit 0, after the +1 (R10).  */
    for (uint64_t i = n; i < L; i++)
        a[i] = 0;
    /* step 5 "Divide the array into 5 partitions: p0, p1, p2, p3, p4"        */
    /* -- contiguous partitions p_k = a[k*P .. (k+1)*P) (R9).                 */
    const uint8_t *p0 = a, *p1 = a + P, *p2 = a + 2 * P, *p3 = a + 3 * P, *p4 = a + 4 * P;
    /* step 6 "Compute a = p0*81 + p1*27 + p2*9 + p3*3 + p4"                  */
#pragma omp parallel for
    for (uint64_t j = 0; j < P; j++)
        out[j] = (uint8_t)(p0[j] * 81 + p1[j] * 27 + p2[j] * 9 + p3[j] * 3 + p4[j]);
    free(a);
}

/* Decoding steps 1-4.  B has P = quartic_len(n) bytes.           */
int tlc_o_quartic_decode(const uint8_t *B, uint64_t P, uint64_t n, int8_t *q)
{
    static const unsigned pow3[5] = {81, 27, 9, 3, 1};
    if (P != tlc_o_quartic_len(n))
        return O_ERR_FORMAT;
    for (uint64_t j = 0; j < P; j++)
        if (B[j] > 242)            /* only 3^5 = 243 codes exist */
            return O_ERR_FORMAT;
    uint64_t L = 5 * P;
    uint8_t *a = (uint8_t *)malloc(L ? L : 1);
    /* step 1 "Restore p0..p4 by dividing a by a power of 3 and taking the    */
    /* remainder"; step 2 "Concatenate p0..p4" -- p_k lands at a[k*P + j].     */
    for (int k = 0; k < 5; k++)
#pragma omp parallel for
        for (uint64_t j = 0; j < P; j++)
            a[(uint64_t)k * P + j] = (uint8_t)((B[j] / pow3[k]) % 3);
    /* step 3 "Unpad, reshape, and type cast"; step 4 "Element-wise subtract 1" */
#pragma omp parallel for
    for (uint64_t i = 0; i < n; i++)
        q[i] = (int8_t)((int)a[i] - 1);
    free(a);
    return O_OK;
}

/* ------------------------------------------------------------------------- */
/* Sec. 3.3 zero-run encoding: "k consecutive occurrences of 121  */
/* (2 <= k <= 14) are replaced with a single byte value of 243+(k-2)".        */
/* Runs longer than 14 are cut greedily into chunks of 14, remainder last     */
/* (R11); a lone 121 stays literal (R12).  Returns the output length.         */
uint64_t tlc_o_zre_encode(const uint8_t *B, uint64_t P, uint8_t *Z)
{
    uint64_t i = 0, z = 0;
    while (i < P) {
        if (B[i] != 121) {
            Z[z++] = B[i++];
            continue;
        }
        uint64_t k = 0;
        while (i + k < P && B[i + k] == 121)
            k++;
        i += k;
        while (k > 0) {
            uint64_t c = k < 14 ? k : 14;
            Z[z++] = (c == 1) ? 121 : (uint8_t)(243 + (c - 2));
            k -= c;
        }
    }
    return z;
}

/* Inverse of zero-run encoding (implied by P:538-548): a byte     */
/* 243+(k-2) expands to k copies of 121, any other byte is itself.  The       */
/* expansion must be exactly P bytes, else FORMAT.                    */
int tlc_o_zre_decode(const uint8_t *Z, uint64_t zlen, uint8_t *B, uint64_t P)
{
    uint64_t o = 0;
    for (uint64_t i = 0; i < zlen; i++) {
        if (Z[i] >= 243) {
            uint64_t k = (uint64_t)(Z[i] - 243) + 2;
            if (o + k > P)
                return O_ERR_FORMAT;
            for (uint64_t r = 0; r < k; r++)
                B[o++] = 121;
        } else {
            if (o + 1 > P)
                return O_ERR_FORMAT;
            B[o++] = Z[i];
        }
    }
    return o == P ? O_OK : O_ERR_FORMAT;
}

/* ------------------------------------------------------------------------- */
/* The whole compressor, Fig. "fig:compression" steps (1),(2),(a),(b),(3),(4) */
/* in that order.  buf (the error-accumulation buffer) is updated  */
/* in place, and left untouched on a data error (R6).                         */
int tlc_o_compress(const float *t, float *buf, uint64_t n, float s, int use_zre,
                   uint8_t *payload, uint64_t cap, float *M_out, uint64_t *len_out)
{
    if (n == 0 || !(s >= 1.0f && s < 2.0f))
        return O_ERR_ARG;
    uint64_t P = tlc_o_quartic_len(n);
    if (cap < P)
        return O_ERR_ARG;
    float *u = (float *)malloc(n * sizeof(float));
    tlc_o_accumulate(t, buf, n, u);                      /* step (1) */
    float M = 0.0f, a = 0.0f;
    int st = tlc_o_scale(u, n, s, &M, &a);               /* Eq. 1    */
    if (st != O_OK) {
        free(u);
        return st;
    }
    int8_t *q = (int8_t *)malloc(n);
    tlc_o_quantize(u, n, M, q);                          /* step (2), Eq. 2 */
    tlc_o_residual(u, q, n, M, buf);                     /* steps (a),(b)   */
    uint8_t *B = (uint8_t *)malloc(P);
    tlc_o_quartic_encode(q, n, B);                       /* step (3)  */
    uint64_t len;
    if (use_zre) {
        len = tlc_o_zre_encode(B, P, payload);           /* step (4)  */
    } else {
        memcpy(payload, B, P);
        len = P;
    }
    *M_out = M;
    *len_out = len;
    free(B);
    free(q);
    free(u);
    return O_OK;
}

/* The decompressor: the compressor's steps reversed.  mode 0     */
/* writes T_out = M*T_q (Eq. 3); mode 1 applies it to out, adding M*q only    */
/* where q != 0 (R16).                                                        */
int tlc_o_decompress(const uint8_t *payload, uint64_t len, int zre_flag, float M,
                     uint64_t n, float *out, int mode)
{
    if (n == 0)
        return O_ERR_ARG;
    /* Eq. 1 makes M = max|T_in| * s a finite (R6) number >= +0: a negative,  */
    /* -0, NaN or infinite M cannot come from the compressor (R21).           */
    if (signbit(M) || !isfinite(M))
        return O_ERR_FORMAT;
    uint64_t P = tlc_o_quartic_len(n);
    uint8_t *B = (uint8_t *)malloc(P);
    int st;
    if (zre_flag) {
        st = tlc_o_zre_decode(payload, len, B, P);
    } else {
        st = (len == P) ? O_OK : O_ERR_FORMAT;
        if (st == O_OK)
            memcpy(B, payload, P);
    }
    if (st != O_OK) {
        free(B);
        return st;
    }
    int8_t *q = (int8_t *)malloc(n);
    st = tlc_o_quartic_decode(B, P, n, q);
    if (st == O_OK) {
        if (mode == 0) {
            tlc_o_dequantize(q, n, M, out);
        } else {
#pragma omp parallel for
            for (uint64_t i = 0; i < n; i++)
                if (q[i] != 0)
                    out[i] = out[i] + M * (float)q[i];
        }
    }
    free(q);
    free(B);
    return st;
}

/* ========================================================================= */
/* Compared designs of Sec. 5.1 that share the 3LC kernels        */
/* (SURVEY 8(f) NEXT-3): "Stoch 3-value + QE" and "8-bit int".  Same rules as */
/* above: fp32, one IEEE operation per source operation, whole-tensor steps.  */
/* ========================================================================= */

/* Philox4x32-10, the counter-based generator of Salmon, Moraes, Dror, Shaw,  */
/* "Parallel random numbers: as easy as 1, 2, 3" (SC'11), Random123 reference:*/
/* ten rounds of                                                              */
/*   (c0,c1,c2,c3) <- (hi(B*c2)^c1^k0, lo(B*c2), hi(A*c0)^c3^k1, lo(A*c0))    */
/* with A = 0xD2511F53, B = 0xCD9E8D57, the key bumped by (0x9E3779B9,        */
/* 0xBB67AE85) after every round.  Pinned by the Random123 known-answer       */
/* vectors (tests/golden/philox_kat.json) and by triton's Philox.             */
void tlc_o_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; r++) {
        uint64_t pa = (uint64_t)0xD2511F53u * c0;
        uint64_t pb = (uint64_t)0xCD9E8D57u * c2;
        uint32_t n0 = (uint32_t)(pb >> 32) ^ c1 ^ k0;
        uint32_t n1 = (uint32_t)pb;
        uint32_t n2 = (uint32_t)(pa >> 32) ^ c3 ^ k1;
        uint32_t n3 = (uint32_t)pa;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* The random word drawn for element e of a tensor at (seed, step) -- reading */
/* R22: word e mod 4 of Philox4x32-10 at counter (e/4 as two 32-bit halves,   */
/* step as two halves) under key (seed low half, seed high half).             */
uint32_t tlc_o_stoch_word(uint64_t seed, uint64_t step, uint64_t e)
{
    uint64_t b = e / 4;
    uint32_t ctr[4] = {(uint32_t)b, (uint32_t)(b >> 32), (uint32_t)step, (uint32_t)(step >> 32)};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t out[4];
    tlc_o_philox4x32_10(ctr, key, out);
    return out[e % 4];
}

/* Stochastic 3-value quantization ("outputs randomized quantization */
/* values whose expectation matches their input value"; "similar to */
/* TernGrad (but without gradient clipping)", no sparsity multiplier and no   */
/* error accumulation buffer).  m = max|t|; element x becomes sign(x) with    */
/* probability |x|/m, else 0.  The draw (R22): U = (w >> 8)*2^-24 */
/* in [0,1) from the element's word w, p = fl(|x| / m), q = sign(x) iff U < p.*/
/* E[m*q] = x up to the 2^-24 grid of U.  m == 0 gives all zeros.             */
int tlc_o_stoch_quantize(const float *t, uint64_t n, uint64_t seed, uint64_t step, int8_t *q, float *m_out)
{
    float m = 0.0f;
    for (uint64_t i = 0; i < n; i++) {
        if (isnan(t[i]) || isinf(t[i]))
            return O_ERR_NONFINITE;
        if (fabsf(t[i]) > m)
            m = fabsf(t[i]);
    }
    for (uint64_t i = 0; i < n; i++) {
        if (m == 0.0f) {
            q[i] = 0;
            continue;
        }
        uint32_t w = tlc_o_stoch_word(seed, step, i);
        float U = (float)(w >> 8) * 0x1p-24f;
        float p = fabsf(t[i]) / m;
        if (U < p)
            q[i] = t[i] > 0.0f ? 1 : -1;
        else
            q[i] = 0;
    }
    *m_out = m;
    return O_OK;
}

/* "Stoch 3-value + QE": the ternary tensor goes through the same */
/* quartic encoding (Sec. 3.2), optionally followed by zero-run encoding; the */
/* receiver decodes it with tlc_o_decompress (M = m).                         */
int tlc_o_stoch_compress(const float *t, uint64_t n, uint64_t seed, uint64_t step, int use_zre,
                         uint8_t *payload, uint64_t cap, float *M_out, uint64_t *len_out)
{
    if (n == 0)
        return O_ERR_ARG;
    uint64_t P = tlc_o_quartic_len(n);
    if (cap < P)
        return O_ERR_ARG;
    int8_t *q = (int8_t *)malloc(n);
    float m = 0.0f;
    int st = tlc_o_stoch_quantize(t, n, seed, step, q, &m);
    if (st != O_OK) {
        free(q);
        return st;
    }
    uint8_t *B = (uint8_t *)malloc(P);
    tlc_o_quartic_encode(q, n, B);
    uint64_t len;
    if (use_zre) {
        len = tlc_o_zre_encode(B, P, payload);
    } else {
        memcpy(payload, B, P);
        len = P;
    }
    *M_out = m;
    *len_out = len;
    free(B);
    free(q);
    return O_OK;
}

/* "8-bit int": "255 distinct values ([-127,127], leaving -128    */
/* unused)".  S:346-354: scale = max|t| / 127 (0 if max = 0), codes =         */
/* round(t / scale) clamped to [-127,127], dequant = scale * code.  round()   */
/* is half away from zero as in Eq. 2 (R1); a scale that underflows to 0 (max */
/* below 127 * 2^-150) gives all-zero codes, like max = 0 (R23).              */
int tlc_o_int8_compress(const float *t, uint64_t n, int8_t *codes, float *scale_out)
{
    if (n == 0)
        return O_ERR_ARG;
    float a = 0.0f;
    for (uint64_t i = 0; i < n; i++) {
        if (isnan(t[i]) || isinf(t[i]))
            return O_ERR_NONFINITE;
        if (fabsf(t[i]) > a)
            a = fabsf(t[i]);
    }
    float scale = a / 127.0f;
    for (uint64_t i = 0; i < n; i++) {
        if (scale == 0.0f) {
            codes[i] = 0;
            continue;
        }
        float c = roundf(t[i] / scale);
        if (c > 127.0f)
            c = 127.0f;
        if (c < -127.0f)
            c = -127.0f;
        codes[i] = (int8_t)c;
    }
    *scale_out = scale;
    return O_OK;
}

/* 8-bit dequantization: mode 0 writes scale * code; mode 1 adds it where     */
/* code != 0 (the accumulate rule R16 of the 3LC decoder).                    */
void tlc_o_int8_decompress(const int8_t *codes, uint64_t n, float scale, float *out, int mode)
{
    for (uint64_t i = 0; i < n; i++) {
        if (mode == 0)
            out[i] = scale * (float)codes[i];
        else if (codes[i] != 0)
            out[i] = out[i] + scale * (float)codes[i];
    }
}
