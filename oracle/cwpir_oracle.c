/*
 * cwpir_oracle.c -- plain-C restatement of the reference server answer path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it.  The product (libcwgpu.so) never links it.
 *
 * It restates, in plain C with 64-bit limbs, the algorithms of
 * /root/reference/proj/core (file:line cited per function).  It is pinned
 * against the compiled reference (oracle/_ref/libcwpir_ref.so) by
 * tests/test_oracle.py and against committed fixtures in tests/golden/.
 *
 * Layouts (same as include/cwgpu.h):
 *   ciphertext [comps][L][N], keys [D][2][L][N] (NTT form), query [h][2][L][N],
 *   db [n][s][N] (< t), positions [n][k] ascending, response [s][2][L][N].
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t u64;
typedef unsigned __int128 u128;

#define ORC_MAXL 8
#define ORC_MAXJ 24
#define ORC_W 28 /* multiword scratch limbs */

/* ---------------- numeric.cpp ---------------- */

static u64 mulmod(u64 a, u64 b, u64 m) { return (u64)(((u128)a * b) % m); }
static u64 addmod(u64 a, u64 b, u64 m) { u64 s = a + b; return (s >= m || s < a) ? s - m : s; }
static u64 submod(u64 a, u64 b, u64 m) { return a >= b ? a - b : a + m - b; }
static u64 negmod(u64 a, u64 m) { return a == 0 ? 0 : m - a; }

/* numeric.cpp:7-16 */
static u64 powmod(u64 b, u64 e, u64 m) {
    u64 r = 1 % m;
    b %= m;
    while (e) {
        if (e & 1) r = mulmod(r, b, m);
        b = mulmod(b, b, m);
        e >>= 1;
    }
    return r;
}

/* numeric.cpp:18-33 (extended Euclid) */
static u64 invmod(u64 a, u64 m) {
    __int128 t = 0, nt = 1, r = m, nr = a % m;
    while (nr) {
        __int128 q = r / nr, tmp = t - q * nt;
        t = nt; nt = tmp;
        tmp = r - q * nr; r = nr; nr = tmp;
    }
    if (t < 0) t += m;
    return (u64)t;
}

/* numeric.cpp:35-61: deterministic Miller-Rabin */
static int is_prime(u64 n) {
    static const u64 W[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return 0;
    for (int i = 0; i < 12; ++i) if (n % W[i] == 0) return n == W[i];
    u64 d = n - 1;
    unsigned s = 0;
    while ((d & 1) == 0) { d >>= 1; ++s; }
    for (int i = 0; i < 12; ++i) {
        u64 x = powmod(W[i], d, n);
        if (x == 1 || x == n - 1) continue;
        int comp = 1;
        for (unsigned j = 1; j < s; ++j) {
            x = mulmod(x, x, n);
            if (x == n - 1) { comp = 0; break; }
        }
        if (comp) return 0;
    }
    return 1;
}

/* numeric.cpp:63-71 */
u64 orc_find_ntt_prime_below(u64 hint, u64 step) {
    u64 p = hint - (hint % step) + 1;
    if (p > hint) p -= step;
    while (p > 3 * step) {
        if (is_prime(p)) return p;
        p -= step;
    }
    return 0;
}

/* numeric.cpp:73-84 */
int orc_find_ntt_primes_below(u64 hint, u64 step, unsigned count, const u64* ex, unsigned nex, u64* out) {
    unsigned got = 0;
    u64 p = hint + 1;
    while (got < count) {
        p = orc_find_ntt_prime_below(p - 1, step);
        if (!p) return -1;
        int skip = 0;
        for (unsigned e = 0; e < nex; ++e) skip |= (ex[e] == p);
        if (!skip) out[got++] = p;
    }
    return 0;
}

/* numeric.cpp:86-108: smallest primitive root */
u64 orc_primitive_root(u64 p) {
    u64 phi = p - 1, n = phi, f[64];
    int nf = 0;
    for (u64 x = 2; x * x <= n; ++x) {
        if (n % x == 0) {
            f[nf++] = x;
            while (n % x == 0) n /= x;
        }
    }
    if (n > 1) f[nf++] = n;
    for (u64 g = 2; g < p; ++g) {
        int ok = 1;
        for (int i = 0; i < nf; ++i) if (powmod(g, phi / f[i], p) == 1) { ok = 0; break; }
        if (ok) return g;
    }
    return 0;
}

/* ---------------- wide.hpp restatement (64-bit limbs) ---------------- */

static void w_clear(u64* a, int n) { memset(a, 0, sizeof(u64) * n); }
static int w_cmp(const u64* a, const u64* b, int n) {
    for (int i = n - 1; i >= 0; --i) if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return 0;
}
static u64 w_sub(u64* a, const u64* b, int n) {
    u64 br = 0;
    for (int i = 0; i < n; ++i) {
        u128 need = (u128)b[i] + br;
        u64 cur = a[i];
        a[i] = cur - (u64)need;
        br = ((u128)cur < need);
    }
    return br;
}
/* wide.hpp:59-73 */
static void w_add_scaled(u64* acc, int nacc, const u64* src, int nsrc, u64 s) {
    u64 c = 0;
    int i = 0;
    for (; i < nsrc; ++i) {
        u128 cur = (u128)src[i] * s + acc[i] + c;
        acc[i] = (u64)cur;
        c = (u64)(cur >> 64);
    }
    for (; c && i < nacc; ++i) {
        u128 x = (u128)acc[i] + c;
        acc[i] = (u64)x;
        c = (u64)(x >> 64);
    }
}
/* n limbs *= s, carry into a[n] (wide.hpp:77-85) */
static void w_mul_u64(u64* a, int n, u64 s) {
    u64 c = 0;
    for (int i = 0; i < n; ++i) {
        u128 cur = (u128)a[i] * s + c;
        a[i] = (u64)cur;
        c = (u64)(cur >> 64);
    }
    a[n] = c;
}
static int w_len(const u64* a, int n) { while (n > 0 && a[n - 1] == 0) --n; return n; }
static int w_bits(const u64* a, int n) {
    n = w_len(a, n);
    if (!n) return 0;
    return 64 * (n - 1) + (64 - __builtin_clzll(a[n - 1]));
}
/* value mod p of a multiword number (bfv.cpp:213-220 computes it with a 2^64-power
 * table; the residue is the same) */
static u64 w_mod(const u64* a, int n, u64 p) {
    u128 r = 0;
    for (int i = n - 1; i >= 0; --i) r = ((r << 64) | a[i]) % p;
    return (u64)r;
}

/* Knuth algorithm D (wide.hpp:176-242): num (nn limbs) / den (nd limbs, top limb != 0).
 * quot gets nn-nd+1 limbs, rem gets nd limbs. */
static void w_divmod(const u64* num, int nn, const u64* den, int nd, u64* quot, u64* rem) {
    u64 u[ORC_W + 2], v[ORC_W];
    nd = w_len(den, nd);
    int sh = __builtin_clzll(den[nd - 1]);
    for (int i = 0; i < nd; ++i) v[i] = (den[i] << sh) | (sh && i ? den[i - 1] >> (64 - sh) : 0);
    u[nn] = sh ? num[nn - 1] >> (64 - sh) : 0;
    for (int i = nn - 1; i >= 0; --i) u[i] = (num[i] << sh) | (sh && i ? num[i - 1] >> (64 - sh) : 0);
    w_clear(quot, nn - nd + 1 > 0 ? nn - nd + 1 : 1);
    if (nn < nd) {
        memcpy(rem, num, 8 * nn);
        for (int i = nn; i < nd; ++i) rem[i] = 0;
        return;
    }
    for (int j = nn - nd; j >= 0; --j) {
        u128 top = ((u128)u[j + nd] << 64) | u[j + nd - 1];
        u128 qhat = top / v[nd - 1];
        u128 rhat = top % v[nd - 1];
        while (qhat >> 64 || (nd >= 2 && qhat * v[nd - 2] > ((rhat << 64) | u[j + nd - 2]))) {
            --qhat;
            rhat += v[nd - 1];
            if (rhat >> 64) break;
        }
        u64 mc = 0, br = 0;
        for (int i = 0; i < nd; ++i) {
            u128 p = (u128)(u64)qhat * v[i] + mc;
            mc = (u64)(p >> 64);
            u128 need = (u128)(u64)p + br;
            u64 cur = u[i + j];
            u[i + j] = cur - (u64)need;
            br = ((u128)cur < need);
        }
        u128 need = (u128)mc + br;
        u64 cur = u[j + nd];
        u[j + nd] = cur - (u64)need;
        if ((u128)cur < need) {
            --qhat;
            u64 c = 0;
            for (int i = 0; i < nd; ++i) {
                u128 s = (u128)u[i + j] + v[i] + c;
                u[i + j] = (u64)s;
                c = (u64)(s >> 64);
            }
            u[j + nd] += c;
        }
        quot[j] = (u64)qhat;
    }
    for (int i = 0; i < nd; ++i) rem[i] = (u[i] >> sh) | (sh ? u[i + 1] << (64 - sh) : 0);
}

/* ---------------- ring.cpp restatement ---------------- */

typedef struct {
    u64 q;
    uint32_t N, logN;
    u64 *rp, *rps, *irp, *irps;
    u64 ninv, ninvs;
} orc_ring;

static unsigned bitrev(unsigned v, unsigned bits) {
    unsigned r = 0;
    for (unsigned i = 0; i < bits; ++i) r = (r << 1) | ((v >> i) & 1);
    return r;
}
static u64 shoup(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }
static u64 mul_shoup_lazy(u64 x, u64 w, u64 ws, u64 q) {
    u64 hi = (u64)(((u128)x * ws) >> 64);
    return x * w - hi * q;
}

/* RingContext::create (ring.cpp:30-74): psi = g^((q-1)/2N), g smallest primitive root,
 * tables indexed by bit-reversed exponent. */
static int ring_init(orc_ring* r, uint32_t N, u64 q) {
    r->q = q;
    r->N = N;
    r->logN = 0;
    while ((1u << r->logN) < N) ++r->logN;
    u64 g = orc_primitive_root(q);
    u64 psi = powmod(g, (q - 1) / (2 * (u64)N), q);
    if (powmod(psi, N, q) != q - 1) return -1;
    u64 psi_inv = invmod(psi, q);
    r->rp = malloc(8 * N); r->rps = malloc(8 * N);
    r->irp = malloc(8 * N); r->irps = malloc(8 * N);
    for (uint32_t i = 0; i < N; ++i) {
        unsigned b = bitrev(i, r->logN);
        r->rp[i] = powmod(psi, b, q);
        r->irp[i] = powmod(psi_inv, b, q);
        r->rps[i] = shoup(r->rp[i], q);
        r->irps[i] = shoup(r->irp[i], q);
    }
    r->ninv = invmod(N % q, q);
    r->ninvs = shoup(r->ninv, q);
    return 0;
}
static void ring_free(orc_ring* r) { free(r->rp); free(r->rps); free(r->irp); free(r->irps); }

/* ring.cpp:78-109 */
static void ntt_fwd(const orc_ring* r, u64* a) {
    const u64 q = r->q, tq = 2 * q;
    const uint32_t n = r->N;
    uint32_t t = n;
    for (uint32_t m = 1; m < n; m <<= 1) {
        t >>= 1;
        for (uint32_t i = 0; i < m; ++i) {
            const u64 w = r->rp[m + i], ws = r->rps[m + i];
            u64* lo = a + 2 * i * t;
            u64* hi = lo + t;
            for (uint32_t j = 0; j < t; ++j) {
                u64 u = lo[j];
                if (u >= tq) u -= tq;
                u64 v = mul_shoup_lazy(hi[j], w, ws, q);
                lo[j] = u + v;
                hi[j] = u - v + tq;
            }
        }
    }
    for (uint32_t j = 0; j < n; ++j) {
        u64 v = a[j];
        if (v >= tq) v -= tq;
        if (v >= q) v -= q;
        a[j] = v;
    }
}
/* ring.cpp:111-144 */
static void ntt_inv(const orc_ring* r, u64* a) {
    const u64 q = r->q, tq = 2 * q;
    const uint32_t n = r->N;
    uint32_t t = 1;
    for (uint32_t m = n; m > 1; m >>= 1) {
        uint32_t h = m >> 1;
        u64* lo = a;
        for (uint32_t i = 0; i < h; ++i) {
            const u64 w = r->irp[h + i], ws = r->irps[h + i];
            u64* hi = lo + t;
            for (uint32_t j = 0; j < t; ++j) {
                u64 u = lo[j], v = hi[j], s = u + v;
                if (s >= tq) s -= tq;
                lo[j] = s;
                hi[j] = mul_shoup_lazy(u - v + tq, w, ws, q);
            }
            lo += 2 * t;
        }
        t <<= 1;
    }
    for (uint32_t j = 0; j < n; ++j) {
        u64 v = mul_shoup_lazy(a[j], r->ninv, r->ninvs, q);
        if (v >= q) v -= q;
        a[j] = v;
    }
}

/* ring.cpp:296-313 */
static void monomial_mul(const u64* a, u64* out, uint32_t n, u64 q, int64_t e) {
    int64_t tn = 2 * (int64_t)n;
    int64_t sh = ((e % tn) + tn) % tn;
    for (uint32_t i = 0; i < n; ++i) {
        u64 pos = i + (u64)sh;
        if (pos < n) out[pos] = a[i];
        else if (pos < 2 * (u64)n) out[pos - n] = negmod(a[i], q);
        else out[pos - 2 * n] = a[i];
    }
}
/* ring.cpp:315-331 */
static void automorphism(const u64* a, u64* out, uint32_t n, u64 q, u64 g) {
    for (uint32_t i = 0; i < n; ++i) {
        u64 e = ((u64)i * g) % (2 * (u64)n);
        if (e < n) out[e] = a[i];
        else out[e - n] = negmod(a[i], q);
    }
}

/* ---------------- BfvContext restatement (bfv.cpp:31-221) ---------------- */

typedef struct {
    uint32_t N, logN, L, J;
    u64 t;
    u64 q[ORC_MAXL], p[ORC_MAXJ];
    orc_ring rq[ORC_MAXL], ra[ORC_MAXJ];
    int q_limbs, p_limbs;
    u64 Q[ORC_W], Qhalf[ORC_W], q_over_qi[ORC_MAXL][ORC_W], mu_q[ORC_MAXL], delta_mod_qi[ORC_MAXL];
    u64 P[ORC_W], Phalf[ORC_W], p_over_pj[ORC_MAXJ][ORC_W], mu_p[ORC_MAXJ];
    unsigned relin_bits, galois_bits, Dr, Dg;
} orc_ctx;

static void big_set_u64(u64* a, u64 v) { w_clear(a, ORC_W); a[0] = v; }
static void big_mul_u64(u64* a, u64 v) { u64 tmp[ORC_W + 1]; memcpy(tmp, a, 8 * ORC_W); w_mul_u64(tmp, ORC_W, v); memcpy(a, tmp, 8 * ORC_W); }
/* a / d for a single-word divisor */
static void big_div_u64(const u64* a, u64 d, u64* out) {
    u128 r = 0;
    for (int i = ORC_W - 1; i >= 0; --i) {
        u128 cur = (r << 64) | a[i];
        out[i] = (u64)(cur / d);
        r = cur % d;
    }
}
static void big_shr1(const u64* a, u64* out) {
    for (int i = 0; i < ORC_W; ++i) out[i] = (a[i] >> 1) | (i + 1 < ORC_W ? a[i + 1] << 63 : 0);
}

static unsigned digit_count(const orc_ctx* c, unsigned bits) {
    if (bits == 0) return c->L;
    return (unsigned)((w_bits(c->Q, ORC_W) + bits - 1) / bits);
}

void orc_free(orc_ctx* c) {
    if (!c) return;
    for (uint32_t i = 0; i < c->L; ++i) ring_free(&c->rq[i]);
    for (uint32_t j = 0; j < c->J; ++j) ring_free(&c->ra[j]);
    free(c);
}

orc_ctx* orc_create(uint32_t N, u64 t, uint32_t L, const u64* primes, unsigned relin_bits, unsigned galois_bits) {
    if (L == 0 || L > ORC_MAXL) return NULL;
    orc_ctx* c = calloc(1, sizeof(orc_ctx));
    c->N = N;
    c->logN = 0;
    while ((1u << c->logN) < N) ++c->logN;
    c->L = L;
    c->t = t;
    big_set_u64(c->Q, 1);
    for (uint32_t i = 0; i < L; ++i) {
        c->q[i] = primes[i];
        if (ring_init(&c->rq[i], N, primes[i])) { orc_free(c); return NULL; }
        big_mul_u64(c->Q, primes[i]);
    }
    c->q_limbs = w_len(c->Q, ORC_W);
    big_shr1(c->Q, c->Qhalf);
    for (uint32_t i = 0; i < L; ++i) {
        big_div_u64(c->Q, c->q[i], c->q_over_qi[i]);
        c->mu_q[i] = invmod(w_mod(c->q_over_qi[i], ORC_W, c->q[i]), c->q[i]);
    }
    u64 delta[ORC_W];
    big_div_u64(c->Q, t, delta);
    for (uint32_t i = 0; i < L; ++i) c->delta_mod_qi[i] = w_mod(delta, ORC_W, c->q[i]);
    /* tensor basis (bfv.cpp:103-123) */
    unsigned need = 2 * w_bits(c->Q, ORC_W) + c->logN + 3;
    unsigned cnt = (need + 58) / 59;
    if (cnt > ORC_MAXJ) { orc_free(c); return NULL; }
    if (orc_find_ntt_primes_below((1ULL << 59) - 1, 2 * (u64)N, cnt, c->q, L, c->p)) { orc_free(c); return NULL; }
    c->J = cnt;
    big_set_u64(c->P, 1);
    for (uint32_t j = 0; j < cnt; ++j) {
        if (ring_init(&c->ra[j], N, c->p[j])) { orc_free(c); return NULL; }
        big_mul_u64(c->P, c->p[j]);
    }
    c->p_limbs = w_len(c->P, ORC_W);
    big_shr1(c->P, c->Phalf);
    for (uint32_t j = 0; j < cnt; ++j) {
        big_div_u64(c->P, c->p[j], c->p_over_pj[j]);
        c->mu_p[j] = invmod(w_mod(c->p_over_pj[j], ORC_W, c->p[j]), c->p[j]);
    }
    c->relin_bits = relin_bits;
    c->galois_bits = galois_bits;
    c->Dr = digit_count(c, relin_bits);
    c->Dg = digit_count(c, galois_bits);
    return c;
}

uint32_t orc_info(const orc_ctx* c, int what) {
    switch (what) {
        case 0: return c->J;
        case 1: return c->Dr;
        case 2: return c->Dg;
        case 3: return (uint32_t)w_bits(c->Q, ORC_W);
        case 4: return (uint32_t)w_bits(c->P, ORC_W);
        default: return 0;
    }
}
u64 orc_aux_prime(const orc_ctx* c, uint32_t j) { return c->p[j]; }

/* crt_q (bfv.cpp:197-209): integer in [0, q) from chain residues; q_limbs+1 limbs */
static void crt_q(const orc_ctx* c, const u64* res, u64* out) {
    const int nl = c->q_limbs + 1;
    w_clear(out, nl);
    for (uint32_t i = 0; i < c->L; ++i) {
        u64 y = mulmod(res[i], c->mu_q[i], c->q[i]);
        w_add_scaled(out, nl, c->q_over_qi[i], c->q_limbs, y);
    }
    while (w_cmp(out, c->Q, nl) >= 0) w_sub(out, c->Q, nl);
}

/* ---------------- BFV server operations ---------------- */

#define LN(c) ((size_t)(c)->L * (c)->N)

void orc_ntt(const orc_ctx* c, int aux, uint32_t idx, u64* a, int inverse) {
    const orc_ring* r = aux ? &c->ra[idx] : &c->rq[idx];
    if (inverse) ntt_inv(r, a); else ntt_fwd(r, a);
}

/* decompose_digits (bfv.cpp:316-339): digits[d][n] */
static void decompose_digits(const orc_ctx* c, const u64* poly, unsigned bits, unsigned D, u64* digits) {
    const uint32_t N = c->N;
    if (bits == 0) {
        for (unsigned d = 0; d < D; ++d) memcpy(digits + (size_t)d * N, poly + (size_t)d * N, 8 * N);
        return;
    }
    const u64 mask = bits == 64 ? ~0ULL : ((1ULL << bits) - 1);
    u64 wide[ORC_W + 1], res[ORC_MAXL];
    for (uint32_t n = 0; n < N; ++n) {
        for (uint32_t i = 0; i < c->L; ++i) res[i] = poly[(size_t)i * N + n];
        crt_q(c, res, wide);
        for (unsigned d = 0; d < D; ++d) {
            unsigned bit = d * bits, limb = bit / 64, off = bit % 64;
            u64 v = wide[limb] >> off;
            if (off && (int)limb + 1 < c->q_limbs + 1) v |= wide[limb + 1] << (64 - off);
            digits[(size_t)d * N + n] = v & mask;
        }
    }
}

/* key_switch (bfv.cpp:343-372): out[2][L][N] coefficient form */
static void key_switch(const orc_ctx* c, const u64* poly, const u64* key, unsigned bits, unsigned D, u64* out) {
    const uint32_t N = c->N, L = c->L;
    u64* dig = malloc(8 * (size_t)D * N);
    u64* dv = malloc(8 * (size_t)N);
    decompose_digits(c, poly, bits, D, dig);
    memset(out, 0, 8 * 2 * LN(c));
    for (unsigned d = 0; d < D; ++d) {
        for (uint32_t i = 0; i < L; ++i) {
            const u64 qi = c->q[i];
            for (uint32_t n = 0; n < N; ++n) {
                u64 v = dig[(size_t)d * N + n];
                dv[n] = v >= qi ? v % qi : v;
            }
            ntt_fwd(&c->rq[i], dv);
            for (int k = 0; k < 2; ++k) {
                const u64* kr = key + (((size_t)d * 2 + k) * L + i) * N;
                u64* acc = out + ((size_t)k * L + i) * N;
                for (uint32_t n = 0; n < N; ++n) acc[n] = addmod(acc[n], mulmod(dv[n], kr[n], qi), qi);
            }
        }
    }
    for (int k = 0; k < 2; ++k)
        for (uint32_t i = 0; i < L; ++i) ntt_inv(&c->rq[i], out + ((size_t)k * L + i) * N);
    free(dig);
    free(dv);
}

/* BfvBackend::substitute (bfv.cpp:694-712) for a 2-component ciphertext */
int orc_substitute(const orc_ctx* c, const u64* ct, u64 g, const u64* gkey, u64* out) {
    const uint32_t N = c->N, L = c->L;
    u64* a1 = malloc(8 * LN(c));
    u64* ks = malloc(8 * 2 * LN(c));
    for (uint32_t i = 0; i < L; ++i) {
        automorphism(ct + (size_t)(L + i) * N, a1 + (size_t)i * N, N, c->q[i], g);
        automorphism(ct + (size_t)i * N, out + (size_t)i * N, N, c->q[i], g);
    }
    key_switch(c, a1, gkey, c->galois_bits, c->Dg, ks);
    for (uint32_t i = 0; i < L; ++i)
        for (uint32_t n = 0; n < N; ++n) {
            size_t o = (size_t)i * N + n;
            out[o] = addmod(out[o], ks[o], c->q[i]);
            out[LN(c) + o] = ks[LN(c) + o];
        }
    free(a1);
    free(ks);
    return 0;
}

/* expand_one / expand_query (expansion.cpp:44-83); galois[a] is the key for g = N/2^a+1 */
int orc_expand(const orc_ctx* c, const u64* query, uint32_t h, uint32_t comp, uint32_t m,
               const u64* galois, u64* out) {
    const uint32_t N = c->N, L = c->L;
    const size_t per = 2 * LN(c), kper = (size_t)c->Dg * 2 * LN(c);
    const size_t chunk = (size_t)1 << comp;
    if ((size_t)h * chunk < m) return -1;
    u64* cts = malloc(8 * per * chunk);
    u64* sub = malloc(8 * per);
    u64* tmp = malloc(8 * per);
    size_t produced = 0;
    for (uint32_t qi = 0; qi < h && produced < m; ++qi) {
        memcpy(cts, query + qi * per, 8 * per);
        for (uint32_t a = 0; a < comp; ++a) {
            const u64 g = N / (1ULL << a) + 1;
            const int64_t shift = -(int64_t)(1ULL << a);
            const size_t level = (size_t)1 << a;
            for (size_t b = 0; b < level; ++b) {
                u64* ctb = cts + b * per;
                u64* ctn = cts + (b + level) * per;
                orc_substitute(c, ctb, g, galois + a * kper, sub);
                for (int k = 0; k < 2; ++k)
                    for (uint32_t i = 0; i < L; ++i) {
                        size_t o = ((size_t)k * L + i) * N;
                        /* shifted - shifted_sub (expansion.cpp:57-58) */
                        monomial_mul(ctb + o, ctn + o, N, c->q[i], shift);
                        monomial_mul(sub + o, tmp + o, N, c->q[i], shift);
                        for (uint32_t n = 0; n < N; ++n) {
                            ctn[o + n] = submod(ctn[o + n], tmp[o + n], c->q[i]);
                            ctb[o + n] = addmod(ctb[o + n], sub[o + n], c->q[i]);
                        }
                    }
            }
        }
        for (size_t j = 0; j < chunk && produced < m; ++j, ++produced)
            memcpy(out + produced * per, cts + j * per, 8 * per);
    }
    free(cts);
    free(sub);
    free(tmp);
    return 0;
}

/* to_aux_basis + aux NTT (bfv.cpp:718-759): prep[2][J][N] */
static void prepare_cipher(const orc_ctx* c, const u64* ct, u64* prep) {
    const uint32_t N = c->N, L = c->L, J = c->J;
    u64 wide[ORC_W + 1], res[ORC_MAXL];
    for (int k = 0; k < 2; ++k) {
        const u64* comp = ct + (size_t)k * LN(c);
        u64* o = prep + (size_t)k * J * N;
        for (uint32_t n = 0; n < N; ++n) {
            for (uint32_t i = 0; i < L; ++i) res[i] = comp[(size_t)i * N + n];
            crt_q(c, res, wide);
            int neg = w_cmp(wide, c->Qhalf, c->q_limbs + 1) > 0;
            if (neg) {
                u64 tmp[ORC_W + 1];
                memcpy(tmp, c->Q, 8 * (c->q_limbs + 1));
                w_sub(tmp, wide, c->q_limbs + 1);
                memcpy(wide, tmp, 8 * (c->q_limbs + 1));
            }
            for (uint32_t j = 0; j < J; ++j) {
                u64 r = w_mod(wide, c->q_limbs + 1, c->p[j]);
                o[(size_t)j * N + n] = neg ? negmod(r, c->p[j]) : r;
            }
        }
        for (uint32_t j = 0; j < J; ++j) ntt_fwd(&c->ra[j], o + (size_t)j * N);
    }
}

/* mul_lazy_prepared (bfv.cpp:765-857) with the exact rounding: out[3][L][N] */
static void mul_lazy_prepared(const orc_ctx* c, const u64* pa, const u64* pb, u64* out) {
    const uint32_t N = c->N, L = c->L, J = c->J;
    u64* d = malloc(8 * 3 * (size_t)J * N);
    for (uint32_t j = 0; j < J; ++j) {
        const u64 p = c->p[j];
        const u64 *a0 = pa + (size_t)j * N, *a1 = pa + (size_t)(J + j) * N;
        const u64 *b0 = pb + (size_t)j * N, *b1 = pb + (size_t)(J + j) * N;
        u64 *d0 = d + (size_t)j * N, *d1 = d + (size_t)(J + j) * N, *d2 = d + (size_t)(2 * J + j) * N;
        for (uint32_t n = 0; n < N; ++n) {
            d0[n] = mulmod(a0[n], b0[n], p);
            d1[n] = addmod(mulmod(a0[n], b1[n], p), mulmod(a1[n], b0[n], p), p);
            d2[n] = mulmod(a1[n], b1[n], p);
        }
        ntt_inv(&c->ra[j], d0);
        ntt_inv(&c->ra[j], d1);
        ntt_inv(&c->ra[j], d2);
    }
    const int acc_limbs = c->p_limbs + 1, mag_limbs = acc_limbs + 1;
    for (int comp = 0; comp < 3; ++comp) {
        for (uint32_t n = 0; n < N; ++n) {
            u64 acc[ORC_W + 2], quot[ORC_W + 2], rem[ORC_W + 2];
            w_clear(acc, mag_limbs + 1);
            for (uint32_t j = 0; j < J; ++j) {
                u64 y = mulmod(d[((size_t)comp * J + j) * N + n], c->mu_p[j], c->p[j]);
                w_add_scaled(acc, acc_limbs, c->p_over_pj[j], c->p_limbs, y);
            }
            while (w_cmp(acc, c->P, acc_limbs) >= 0) w_sub(acc, c->P, acc_limbs);
            int neg = w_cmp(acc, c->Phalf, acc_limbs) > 0;
            if (neg) {
                u64 tmp[ORC_W + 2];
                memcpy(tmp, c->P, 8 * acc_limbs);
                w_sub(tmp, acc, acc_limbs);
                memcpy(acc, tmp, 8 * acc_limbs);
            }
            w_mul_u64(acc, acc_limbs, c->t);
            /* floor division by q; round half up on the magnitude (exact form of
             * bfv.cpp:832-842, rem[q_limbs] zeroed) */
            w_divmod(acc, mag_limbs, c->Q, c->q_limbs, quot, rem);
            u64 r2[ORC_W + 1];
            memcpy(r2, rem, 8 * c->q_limbs);
            r2[c->q_limbs] = 0;
            /* 2*rem >= q */
            u64 carry = 0;
            for (int l = 0; l <= c->q_limbs; ++l) {
                u64 nv = (r2[l] << 1) | carry;
                carry = r2[l] >> 63;
                r2[l] = nv;
            }
            u64 qpad[ORC_W + 1];
            memcpy(qpad, c->Q, 8 * (c->q_limbs + 1));
            qpad[c->q_limbs] = 0;
            const int ql = mag_limbs - c->q_limbs + 1;
            if (w_cmp(r2, qpad, c->q_limbs + 1) >= 0) {
                for (int l = 0; l < ql; ++l) if (++quot[l]) break;
            }
            for (uint32_t i = 0; i < L; ++i) {
                u64 r = w_mod(quot, ql, c->q[i]);
                out[((size_t)comp * L + i) * N + n] = neg ? negmod(r, c->q[i]) : r;
            }
        }
    }
    free(d);
}

/* relinearize (bfv.cpp:859-869): ct3 -> ct2 */
int orc_relinearize(const orc_ctx* c, const u64* ct3, const u64* relin, u64* out) {
    const uint32_t N = c->N, L = c->L;
    u64* ks = malloc(8 * 2 * LN(c));
    key_switch(c, ct3 + 2 * LN(c), relin, c->relin_bits, c->Dr, ks);
    for (int k = 0; k < 2; ++k)
        for (uint32_t i = 0; i < L; ++i)
            for (uint32_t n = 0; n < N; ++n) {
                size_t o = ((size_t)k * L + i) * N + n;
                out[o] = addmod(ct3[o], ks[o], c->q[i]);
            }
    free(ks);
    return 0;
}

/* mul_lazy on two ciphertexts (a 3-component operand is finalized first, bfv.cpp:750) */
int orc_mul_lazy(const orc_ctx* c, const u64* a, uint32_t ca, const u64* b, uint32_t cb,
                 const u64* relin, u64* out) {
    const size_t pj = 2 * (size_t)c->J * c->N;
    u64* pa = malloc(8 * pj);
    u64* pb = malloc(8 * pj);
    u64* tmp = malloc(8 * 2 * LN(c));
    if (ca == 3) { orc_relinearize(c, a, relin, tmp); prepare_cipher(c, tmp, pa); } else prepare_cipher(c, a, pa);
    if (cb == 3) { orc_relinearize(c, b, relin, tmp); prepare_cipher(c, tmp, pb); } else prepare_cipher(c, b, pb);
    mul_lazy_prepared(c, pa, pb, out);
    free(pa); free(pb); free(tmp);
    return 0;
}

/* mul = relinearize(mul_lazy) (bfv.cpp:877-879) */
int orc_mul(const orc_ctx* c, const u64* a, const u64* b, const u64* relin, u64* out) {
    u64* t3 = malloc(8 * 3 * LN(c));
    orc_mul_lazy(c, a, 2, b, 2, relin, t3);
    orc_relinearize(c, t3, relin, out);
    free(t3);
    return 0;
}

/* product_tree (eq_circuits.cpp:53-69) over `cnt` ciphertexts of comps[i] components.
 * nodes are [3][L][N] slots; result written into out, its comps returned. */
static uint32_t product_tree(const orc_ctx* c, u64* nodes, uint32_t* comps, uint32_t cnt, int lazy_root,
                             const u64* relin, u64* out) {
    const size_t slot = 3 * LN(c);
    while (cnt > 1) {
        int last = cnt == 2;
        uint32_t nn = 0;
        for (uint32_t i = 0; i + 1 < cnt; i += 2) {
            u64* dst = malloc(8 * slot);
            if (last && lazy_root) {
                orc_mul_lazy(c, nodes + i * slot, comps[i], nodes + (i + 1) * slot, comps[i + 1], relin, dst);
                comps[nn] = 3;
            } else {
                u64* t3 = malloc(8 * slot);
                orc_mul_lazy(c, nodes + i * slot, comps[i], nodes + (i + 1) * slot, comps[i + 1], relin, t3);
                orc_relinearize(c, t3, relin, dst);
                free(t3);
                comps[nn] = 2;
            }
            memcpy(nodes + nn * slot, dst, 8 * slot);
            free(dst);
            ++nn;
        }
        if (cnt % 2) {
            memmove(nodes + nn * slot, nodes + (cnt - 1) * slot, 8 * slot);
            comps[nn] = comps[cnt - 1];
            ++nn;
        }
        cnt = nn;
    }
    memcpy(out, nodes, 8 * comps[0] * LN(c));
    return comps[0];
}

/* selection ciphertext of one row (pir.cpp:287-302 / SURVEY A12). sel is [3][L][N];
 * returns its component count. prep = prepared entries [m][2][J][N] (op 0, k>=2). */
static uint32_t select_row(const orc_ctx* c, const u64* expanded, const u64* prep, const uint32_t* pos,
                           uint32_t k, uint32_t op, const u64* relin, u64* sel) {
    const size_t per = 2 * LN(c), slot = 3 * LN(c), pj = 2 * (size_t)c->J * c->N;
    const uint32_t N = c->N, L = c->L;
    if (op == 0) {
        if (k == 1) { memcpy(sel, expanded + pos[0] * per, 8 * per); return 2; }
        uint32_t cnt = 0, comps[64];
        u64* nodes = malloc(8 * slot * (k / 2 + 1));
        for (uint32_t p = 0; p + 1 < k; p += 2) {
            u64* dst = nodes + cnt * slot;
            if (k == 2) {
                mul_lazy_prepared(c, prep + pos[p] * pj, prep + pos[p + 1] * pj, dst);
                comps[cnt++] = 3;
            } else {
                u64* t3 = malloc(8 * slot);
                mul_lazy_prepared(c, prep + pos[p] * pj, prep + pos[p + 1] * pj, t3);
                orc_relinearize(c, t3, relin, dst);
                free(t3);
                comps[cnt++] = 2;
            }
        }
        if (k % 2) { memcpy(nodes + cnt * slot, expanded + pos[k - 1] * per, 8 * per); comps[cnt++] = 2; }
        uint32_t r = product_tree(c, nodes, comps, cnt, 1, relin, sel);
        free(nodes);
        return r;
    }
    /* arithmetic operator */
    const u64 t = c->t;
    u64 f = 1;
    for (uint32_t i = 2; i <= k; ++i) f = mulmod(f, i % t, t);
    const u64 kinv = invmod(f, t);
    u64* nodes = malloc(8 * slot * k);
    uint32_t comps[64];
    u64* inner = nodes; /* factor 0 */
    memcpy(inner, expanded + pos[0] * per, 8 * per);
    for (uint32_t p = 1; p < k; ++p) {
        const u64* e = expanded + pos[p] * per;
        for (uint32_t x = 0; x < 2 * L; ++x) {
            u64 qi = c->q[x % L];
            for (uint32_t n = 0; n < N; ++n) inner[(size_t)x * N + n] = addmod(inner[(size_t)x * N + n], e[(size_t)x * N + n], qi);
        }
    }
    comps[0] = 2;
    for (uint32_t fi = 1; fi < k; ++fi) {
        u64* fdst = nodes + fi * slot;
        memcpy(fdst, inner, 8 * per);
        /* add_plain(inner, t - fi) -> c0 += Delta * (t - fi) (bfv.cpp:641-649, 267-274) */
        u64 mval = t - (fi % t);
        for (uint32_t i = 0; i < L; ++i) fdst[(size_t)i * N] = addmod(fdst[(size_t)i * N], mulmod(c->delta_mod_qi[i], mval % c->q[i], c->q[i]), c->q[i]);
        comps[fi] = 2;
    }
    uint32_t r = product_tree(c, nodes, comps, k, 0, relin, sel);
    /* plain_mul by the constant (k!)^-1 mod t (bfv.cpp:664-680) */
    for (uint32_t x = 0; x < r * L; ++x) {
        u64 qi = c->q[x % L];
        for (uint32_t n = 0; n < N; ++n) sel[(size_t)x * N + n] = mulmod(sel[(size_t)x * N + n], kinv % qi, qi);
    }
    free(nodes);
    return r;
}

/* Full server answer (pir.cpp:337-347 composed as in oracle/ref_harness.cpp:ref_answer).
 * galois: [comp][Dg][2][L][N] for a = 0..comp-1. out: [s][2][L][N]. */
int orc_answer(const orc_ctx* c, const u64* relin, const u64* galois, const u64* query, uint32_t h,
               uint32_t comp, uint32_t m, uint64_t n, uint32_t k, const uint32_t* positions, uint32_t s,
               const u64* db, uint32_t op, u64* out) {
    const uint32_t N = c->N, L = c->L;
    const size_t per = 2 * LN(c), pj = 2 * (size_t)c->J * N;
    u64* expanded = malloc(8 * per * m);
    if (orc_expand(c, query, h, comp, m, galois, expanded)) { free(expanded); return -1; }
    u64* prep = NULL;
    if (op == 0 && k >= 2) {
        prep = malloc(8 * pj * m);
        for (uint32_t j = 0; j < m; ++j) prepare_cipher(c, expanded + j * per, prep + j * pj);
    }
    /* acc[s][3][L][N] NTT-domain (weighted_sum, bfv.cpp:944-986) */
    u64* acc = calloc(3 * LN(c) * s, 8);
    u64* sel = malloc(8 * 3 * LN(c));
    u64* tmp = malloc(8 * N);
    u64* pl = malloc(8 * N);
    uint32_t nc = 0;
    for (uint64_t r = 0; r < n; ++r) {
        uint32_t sc = select_row(c, expanded, prep, positions + r * k, k, op, relin, sel);
        if (sc > nc) nc = sc;
        for (uint32_t j = 0; j < s; ++j) {
            for (uint32_t i = 0; i < L; ++i) {
                memcpy(pl, db + (r * s + j) * N, 8 * N);
                for (uint32_t x = 0; x < N; ++x) pl[x] %= c->q[i];
                ntt_fwd(&c->rq[i], pl);
                for (uint32_t kk = 0; kk < sc; ++kk) {
                    memcpy(tmp, sel + ((size_t)kk * L + i) * N, 8 * N);
                    ntt_fwd(&c->rq[i], tmp);
                    u64* a = acc + (((size_t)j * 3 + kk) * L + i) * N;
                    for (uint32_t x = 0; x < N; ++x) a[x] = addmod(a[x], mulmod(tmp[x], pl[x], c->q[i]), c->q[i]);
                }
            }
        }
    }
    u64* r3 = malloc(8 * 3 * LN(c));
    for (uint32_t j = 0; j < s; ++j) {
        memcpy(r3, acc + (size_t)j * 3 * LN(c), 8 * 3 * LN(c));
        for (uint32_t kk = 0; kk < nc; ++kk)
            for (uint32_t i = 0; i < L; ++i) ntt_inv(&c->rq[i], r3 + ((size_t)kk * L + i) * N);
        if (nc == 3) orc_relinearize(c, r3, relin, out + j * per);
        else memcpy(out + j * per, r3, 8 * per);
    }
    free(r3); free(acc); free(sel); free(tmp); free(pl); free(prep); free(expanded);
    return 0;
}

/* The selection vector alone (config 2): sel[n][3][L][N] (2-comp rows zero-padded);
 * comps_out[n] receives each row's component count. */
int orc_select(const orc_ctx* c, const u64* relin, const u64* galois, const u64* query, uint32_t h,
               uint32_t comp, uint32_t m, uint64_t n, uint32_t k, const uint32_t* positions, uint32_t op,
               u64* sel, uint32_t* comps_out) {
    const size_t per = 2 * LN(c), pj = 2 * (size_t)c->J * c->N;
    u64* expanded = malloc(8 * per * m);
    if (orc_expand(c, query, h, comp, m, galois, expanded)) { free(expanded); return -1; }
    u64* prep = NULL;
    if (op == 0 && k >= 2) {
        prep = malloc(8 * pj * m);
        for (uint32_t j = 0; j < m; ++j) prepare_cipher(c, expanded + j * per, prep + j * pj);
    }
    for (uint64_t r = 0; r < n; ++r) {
        u64* dst = sel + r * 3 * LN(c);
        memset(dst, 0, 8 * 3 * LN(c));
        comps_out[r] = select_row(c, expanded, prep, positions + r * k, k, op, relin, dst);
    }
    free(prep);
    free(expanded);
    return 0;
}
