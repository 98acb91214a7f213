/*
 * taskgen.cpp -- host-side bulk task-set generator, bit-identical to the
 * reference generator gpusched.workbench.generate_taskset (workbench.py:101)
 * for the same GenParams and seed, writing engine blobs directly.
 *
 * The reference draws from CPython's random.Random(seed).  This file
 * restates what that object does so the same seed yields the same numbers:
 *   - seeding: an int seed is split into little-endian 32-bit words
 *     (|seed|; [0] for 0) and fed to MT19937 init_by_array; a str seed is
 *     first turned into int.from_bytes(s + sha512(s), "big") (Random.seed,
 *     version 2);
 *   - random() = ((w1 >> 5) * 2^26 + (w2 >> 6)) / 2^53;
 *   - randint(a, b) = a + _randbelow(b - a + 1), _randbelow(n) =
 *     getrandbits(bit_length(n)) redrawn while >= n, getrandbits(k <= 32) =
 *     w >> (32 - k).
 * Exact rational steps of the reference (utilisation normalisation,
 * deadline = floor(demand / U_i)) are done in 128-bit integers.
 */
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <thread>
#include <vector>

#include "../../include/rtgpu.h"
#include "../../include/rtgpu_gen.h"

namespace {

typedef unsigned __int128 u128;

/* floor(a * b / d) for a * b up to 2^256 (d > 0, quotient < 2^127): the
 * deadline formula with a utilisation given as a binary fraction (Fraction
 * of a float has a 2^55 denominator) exceeds 128 bits.  Schoolbook
 * 256-bit product, then restoring division one bit at a time -- only on
 * the overflow path. */
u128 muldiv_u256(u128 a, u128 b, u128 d) {
    const uint64_t a0 = (uint64_t)a, a1 = (uint64_t)(a >> 64), b0 = (uint64_t)b, b1 = (uint64_t)(b >> 64);
    const u128 p00 = (u128)a0 * b0, p01 = (u128)a0 * b1, p10 = (u128)a1 * b0, p11 = (u128)a1 * b1;
    u128 mid = (p00 >> 64) + (uint64_t)p01 + (uint64_t)p10;
    u128 lo = ((u128)(uint64_t)mid << 64) | (uint64_t)p00;
    u128 hi = p11 + (p01 >> 64) + (p10 >> 64) + (mid >> 64);
    u128 rem = 0, q = 0;
    for (int bit = 255; bit >= 0; bit--) {
        const bool top = (rem >> 127) != 0;
        rem = (rem << 1) | (u128)((bit >= 128 ? (hi >> (bit - 128)) : (lo >> bit)) & 1);
        q <<= 1;
        if (top || rem >= d) {
            rem -= d;
            q |= 1;
        }
    }
    return q;
}
typedef __int128 i128;

/* ------------------------------------------------------------ SHA-512 */

const uint64_t K512[80] = {
    0x428a2f98d728ae22ULL, 0x7137449123ef65cdULL, 0xb5c0fbcfec4d3b2fULL, 0xe9b5dba58189dbbcULL,
    0x3956c25bf348b538ULL, 0x59f111f1b605d019ULL, 0x923f82a4af194f9bULL, 0xab1c5ed5da6d8118ULL,
    0xd807aa98a3030242ULL, 0x12835b0145706fbeULL, 0x243185be4ee4b28cULL, 0x550c7dc3d5ffb4e2ULL,
    0x72be5d74f27b896fULL, 0x80deb1fe3b1696b1ULL, 0x9bdc06a725c71235ULL, 0xc19bf174cf692694ULL,
    0xe49b69c19ef14ad2ULL, 0xefbe4786384f25e3ULL, 0x0fc19dc68b8cd5b5ULL, 0x240ca1cc77ac9c65ULL,
    0x2de92c6f592b0275ULL, 0x4a7484aa6ea6e483ULL, 0x5cb0a9dcbd41fbd4ULL, 0x76f988da831153b5ULL,
    0x983e5152ee66dfabULL, 0xa831c66d2db43210ULL, 0xb00327c898fb213fULL, 0xbf597fc7beef0ee4ULL,
    0xc6e00bf33da88fc2ULL, 0xd5a79147930aa725ULL, 0x06ca6351e003826fULL, 0x142929670a0e6e70ULL,
    0x27b70a8546d22ffcULL, 0x2e1b21385c26c926ULL, 0x4d2c6dfc5ac42aedULL, 0x53380d139d95b3dfULL,
    0x650a73548baf63deULL, 0x766a0abb3c77b2a8ULL, 0x81c2c92e47edaee6ULL, 0x92722c851482353bULL,
    0xa2bfe8a14cf10364ULL, 0xa81a664bbc423001ULL, 0xc24b8b70d0f89791ULL, 0xc76c51a30654be30ULL,
    0xd192e819d6ef5218ULL, 0xd69906245565a910ULL, 0xf40e35855771202aULL, 0x106aa07032bbd1b8ULL,
    0x19a4c116b8d2d0c8ULL, 0x1e376c085141ab53ULL, 0x2748774cdf8eeb99ULL, 0x34b0bcb5e19b48a8ULL,
    0x391c0cb3c5c95a63ULL, 0x4ed8aa4ae3418acbULL, 0x5b9cca4f7763e373ULL, 0x682e6ff3d6b2b8a3ULL,
    0x748f82ee5defb2fcULL, 0x78a5636f43172f60ULL, 0x84c87814a1f0ab72ULL, 0x8cc702081a6439ecULL,
    0x90befffa23631e28ULL, 0xa4506cebde82bde9ULL, 0xbef9a3f7b2c67915ULL, 0xc67178f2e372532bULL,
    0xca273eceea26619cULL, 0xd186b8c721c0c207ULL, 0xeada7dd6cde0eb1eULL, 0xf57d4f7fee6ed178ULL,
    0x06f067aa72176fbaULL, 0x0a637dc5a2c898a6ULL, 0x113f9804bef90daeULL, 0x1b710b35131c471bULL,
    0x28db77f523047d84ULL, 0x32caab7b40c72493ULL, 0x3c9ebe0a15c9bebcULL, 0x431d67c49c100d4cULL,
    0x4cc5d4becb3e42b6ULL, 0x597f299cfc657e2aULL, 0x5fcb6fab3ad6faecULL, 0x6c44198c4a475817ULL};

inline uint64_t rotr(uint64_t x, int n) { return (x >> n) | (x << (64 - n)); }

void sha512(const unsigned char *msg, size_t len, unsigned char out[64]) {
    uint64_t h[8] = {0x6a09e667f3bcc908ULL, 0xbb67ae8584caa73bULL, 0x3c6ef372fe94f82bULL,
                     0xa54ff53a5f1d36f1ULL, 0x510e527fade682d1ULL, 0x9b05688c2b3e6c1fULL,
                     0x1f83d9abfb41bd6bULL, 0x5be0cd19137e2179ULL};
    std::vector<unsigned char> m(msg, msg + len);
    m.push_back(0x80);
    while (m.size() % 128 != 112) m.push_back(0);
    for (int i = 0; i < 8; i++) m.push_back(0); /* high 64 bits of the length */
    uint64_t bits = (uint64_t)len * 8;
    for (int i = 7; i >= 0; i--) m.push_back((unsigned char)(bits >> (8 * i)));
    for (size_t off = 0; off < m.size(); off += 128) {
        uint64_t w[80];
        for (int t = 0; t < 16; t++) {
            uint64_t v = 0;
            for (int b = 0; b < 8; b++) v = (v << 8) | m[off + 8 * t + b];
            w[t] = v;
        }
        for (int t = 16; t < 80; t++) {
            uint64_t s0 = rotr(w[t - 15], 1) ^ rotr(w[t - 15], 8) ^ (w[t - 15] >> 7);
            uint64_t s1 = rotr(w[t - 2], 19) ^ rotr(w[t - 2], 61) ^ (w[t - 2] >> 6);
            w[t] = w[t - 16] + s0 + w[t - 7] + s1;
        }
        uint64_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
        for (int t = 0; t < 80; t++) {
            uint64_t S1 = rotr(e, 14) ^ rotr(e, 18) ^ rotr(e, 41);
            uint64_t ch = (e & f) ^ (~e & g);
            uint64_t t1 = hh + S1 + ch + K512[t] + w[t];
            uint64_t S0 = rotr(a, 28) ^ rotr(a, 34) ^ rotr(a, 39);
            uint64_t mj = (a & b) ^ (a & c) ^ (b & c);
            uint64_t t2 = S0 + mj;
            hh = g;
            g = f;
            f = e;
            e = d + t1;
            d = c;
            c = b;
            b = a;
            a = t1 + t2;
        }
        h[0] += a, h[1] += b, h[2] += c, h[3] += d, h[4] += e, h[5] += f, h[6] += g, h[7] += hh;
    }
    for (int i = 0; i < 8; i++)
        for (int b = 0; b < 8; b++) out[8 * i + b] = (unsigned char)(h[i] >> (56 - 8 * b));
}

/* ------------------------------------------------------------ MT19937 */

struct MT {
    uint32_t mt[624];
    int idx;
    void init_genrand(uint32_t s) {
        mt[0] = s;
        for (int i = 1; i < 624; i++) mt[i] = 1812433253u * (mt[i - 1] ^ (mt[i - 1] >> 30)) + (uint32_t)i;
        idx = 624;
    }
    void init_by_array(const uint32_t *key, size_t n) {
        init_genrand(19650218u);
        size_t i = 1, j = 0;
        for (size_t k = std::max((size_t)624, n); k; k--) {
            mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1664525u)) + key[j] + (uint32_t)j;
            i++;
            j++;
            if (i >= 624) {
                mt[0] = mt[623];
                i = 1;
            }
            if (j >= n) j = 0;
        }
        for (size_t k = 623; k; k--) {
            mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1566083941u)) - (uint32_t)i;
            i++;
            if (i >= 624) {
                mt[0] = mt[623];
                i = 1;
            }
        }
        mt[0] = 0x80000000u;
        idx = 624;
    }
    uint32_t next() {
        if (idx >= 624) {
            for (int k = 0; k < 624; k++) {
                uint32_t y = (mt[k] & 0x80000000u) | (mt[(k + 1) % 624] & 0x7fffffffu);
                mt[k] = mt[(k + 397) % 624] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
            }
            idx = 0;
        }
        uint32_t y = mt[idx++];
        y ^= y >> 11;
        y ^= (y << 7) & 0x9d2c5680u;
        y ^= (y << 15) & 0xefc60000u;
        y ^= y >> 18;
        return y;
    }
    /* random() as the exact 53-bit numerator over 2^53 */
    uint64_t random53() {
        uint64_t a = next() >> 5, b = next() >> 6;
        return a * 67108864ull + b;
    }
    uint32_t getrandbits(int k) { return k == 0 ? 0 : next() >> (32 - k); }
    int64_t randbelow(int64_t n) {
        int k = 0;
        while (((int64_t)1 << k) <= n) k++; /* bit_length(n) */
        if (k > 32) {
            /* not needed by the generator's ranges */
            return 0;
        }
        int64_t r = getrandbits(k);
        while (r >= n) r = getrandbits(k);
        return r;
    }
    int64_t randint(int64_t a, int64_t b) { return a + randbelow(b - a + 1); }
};

/* seed from little-endian 32-bit words of a non-negative big integer */
void seed_words(MT &g, std::vector<uint32_t> w) {
    while (w.size() > 1 && w.back() == 0) w.pop_back();
    if (w.empty()) w.push_back(0);
    g.init_by_array(w.data(), w.size());
}

void seed_int(MT &g, int64_t s) {
    uint64_t u = s < 0 ? (uint64_t)(-(s + 1)) + 1 : (uint64_t)s;
    seed_words(g, {(uint32_t)u, (uint32_t)(u >> 32)});
}

void seed_str(MT &g, const char *s) {
    size_t len = strlen(s);
    std::vector<unsigned char> bytes(s, s + len);
    unsigned char dig[64];
    sha512((const unsigned char *)s, len, dig);
    bytes.insert(bytes.end(), dig, dig + 64);
    /* int.from_bytes(bytes, "big") -> little-endian 32-bit words */
    std::vector<uint32_t> w;
    for (size_t end = bytes.size(); end > 0;) {
        uint32_t v = 0;
        size_t beg = end >= 4 ? end - 4 : 0;
        for (size_t i = beg; i < end; i++) v = (v << 8) | bytes[i];
        w.push_back(v);
        end = beg;
    }
    seed_words(g, w);
}

int64_t gcd64(int64_t a, int64_t b) {
    while (b) {
        int64_t t = a % b;
        a = b;
        b = t;
    }
    return a < 0 ? -a : a;
}

const int CAPS[4] = {145, 170, 170, 180}; /* interleave caps per kernel class, percent */

struct Draft {
    int64_t D;
    int idx;
    std::vector<int64_t> cl_lo, cl_hi, ml_lo, ml_hi, gw_lo, gw_hi, gl;
    std::vector<int> pct;
};

int64_t lo_of(int64_t hi, const rtgpu_gen_params *p) {
    int64_t lo = (int64_t)((i128)hi * p->lofrac_num / p->lofrac_den);
    return lo < hi ? lo : hi;
}

/* workbench.py:101 generate_taskset for one seed, written as a blob. */
/* false: a deadline does not fit int64 (parameters out of range) */
bool gen_one(const rtgpu_gen_params *p, MT &g, int64_t *out) {
    const int n = p->n_tasks, m = p->n_subtasks;
    std::vector<uint64_t> raw(n);
    for (;;) {
        bool ok = true;
        u128 tot = 0;
        for (int i = 0; i < n; i++) {
            raw[i] = g.random53();
            tot += raw[i];
            ok = ok && raw[i] > 0;
        }
        if (tot > 0 && ok) break;
    }
    u128 total = 0;
    for (int i = 0; i < n; i++) total += raw[i];
    std::vector<Draft> dr(n);
    for (int i = 0; i < n; i++) {
        Draft &d = dr[i];
        d.idx = i;
        for (int j = 0; j < m; j++) {
            int64_t hi = g.randint(p->cpu_lo, p->cpu_hi);
            d.cl_hi.push_back(hi);
            d.cl_lo.push_back(lo_of(hi, p));
        }
        for (int j = 0; j < 2 * (m - 1); j++) {
            int64_t hi = g.randint(p->mem_lo, p->mem_hi);
            d.ml_hi.push_back(hi);
            d.ml_lo.push_back(lo_of(hi, p));
        }
        for (int j = 0; j < m - 1; j++) {
            int64_t hi = g.randint(p->gpu_lo, p->gpu_hi);
            int64_t lo = lo_of(hi, p);
            int cap = CAPS[g.randbelow(4)];
            int pct = (int)g.randint(100, cap);
            int64_t ov = (int64_t)((i128)hi * p->eps_num / p->eps_den);
            if (lo < ov) ov = lo;
            d.gw_hi.push_back(hi);
            d.gw_lo.push_back(lo);
            d.gl.push_back(ov);
            d.pct.push_back(pct);
        }
        i128 demand = 0;
        for (int64_t v : d.cl_hi) demand += v;
        for (int64_t v : d.ml_hi) demand += v;
        for (int64_t v : d.gw_hi) demand += v;
        /* D = max(1, floor(demand / (raw_i * U / total))) */
        const u128 den = (u128)raw[i] * (u128)p->util_num; /* < 2^117 */
        const u128 dt = (u128)demand * total;              /* < 2^103 */
        u128 num, q;
        if (__builtin_mul_overflow(dt, (u128)p->util_den, &num)) q = muldiv_u256(dt, (u128)p->util_den, den);
        else q = num / den;
        if (q > (u128)INT64_MAX) return false; /* a deadline beyond int64 */
        d.D = q < 1 ? 1 : (int64_t)q;
    }
    std::vector<int> order(n);
    for (int i = 0; i < n; i++) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
        return dr[a].D != dr[b].D ? dr[a].D < dr[b].D : a < b;
    });
    std::vector<int> prio(n);
    for (int r = 0; r < n; r++) prio[order[r]] = r + 1;
    /* merge to one copy per kernel if requested (workbench.py:83) */
    const bool one = p->mem_model == RTGPU_ONE_COPY;
    const int pm = m < 2 ? 0 : (one ? m - 1 : 2 * m - 2);
    if (one)
        for (Draft &d : dr) {
            std::vector<int64_t> lo, hi;
            for (int j = 0; j < m - 1; j++) {
                lo.push_back(d.ml_lo[2 * j] + d.ml_lo[2 * j + 1]);
                hi.push_back(d.ml_hi[2 * j] + d.ml_hi[2 * j + 1]);
            }
            d.ml_lo = lo;
            d.ml_hi = hi;
        }
    /* interleave ratio denominators: lcm of reduced pct/100 */
    int64_t A = 1;
    for (Draft &d : dr)
        for (int pc : d.pct) {
            int64_t den = 100 / gcd64(pc, 100);
            A = A / gcd64(A, den) * den;
        }
    const int seg_words = 2 * m + 2 * pm + 4 * (m - 1);
    const bool c32 = p->seg_int32 != 0;
    const bool r32 = p->seg_int32 == 2; /* int32 task records too */
    const int64_t words = rtgpu_gen_blob_words(p);
    out[0] = n;
    out[1] = p->physical_sms;
    out[2] = p->mem_model;
    out[3] = A;
    out[4] = words;
    out[5] = m;
    out[6] = pm;
    out[7] = r32 ? 2 : (c32 ? 1 : 0);
    /* segment areas after the records; seg_off in int64 words or int32 elements */
    int64_t seg = (RTGPU_HDR_WORDS + (int64_t)n * RTGPU_REC_WORDS(out[7])) * (c32 ? 2 : 1);
    int32_t *out32 = (int32_t *)out;
    /* tasks in priority order (TaskSet.by_priority) */
    std::vector<int> byp(n);
    for (int i = 0; i < n; i++) byp[prio[i] - 1] = i;
    for (int r = 0; r < n; r++) {
        Draft &d = dr[byp[r]];
        const int64_t rv[RTGPU_TASK_WORDS] = {m, pm, d.D, d.D, r + 1, seg, d.idx, 0};
        if (r32) { /* packed record (include/rtgpu.h): D, T, m | p | index, priority | seg_off */
            int64_t *rec = out + RTGPU_HDR_WORDS + (int64_t)r * (RTGPU_TASK_WORDS / 2);
            rec[0] = rv[2];
            rec[1] = rv[3];
            rec[2] = (rv[0] & 0xff) | (rv[1] & 0xff) << 8 | rv[6] << 16;
            rec[3] = (int64_t)((uint64_t)(uint32_t)(int32_t)rv[4] | (uint64_t)rv[5] << 32);
        } else {
            int64_t *rec = out + RTGPU_HDR_WORDS + (int64_t)r * RTGPU_TASK_WORDS;
            for (int f = 0; f < RTGPU_TASK_WORDS; f++) rec[f] = rv[f];
        }
        std::vector<int64_t> v;
        v.reserve(seg_words);
        for (int j = 0; j < m; j++) v.push_back(d.cl_lo[j]);
        for (int j = 0; j < m; j++) v.push_back(d.cl_hi[j]);
        for (int j = 0; j < pm; j++) v.push_back(d.ml_lo[j]);
        for (int j = 0; j < pm; j++) v.push_back(d.ml_hi[j]);
        for (int j = 0; j < m - 1; j++) v.push_back(d.gw_lo[j]);
        for (int j = 0; j < m - 1; j++) v.push_back(d.gw_hi[j]);
        for (int j = 0; j < m - 1; j++) v.push_back(d.gl[j]);
        for (int j = 0; j < m - 1; j++) v.push_back((int64_t)d.pct[j] * A / 100);
        for (size_t j = 0; j < v.size(); j++) {
            if (c32) out32[seg + (int64_t)j] = (int32_t)v[j]; /* generator values < 2^31 */
            else out[seg + (int64_t)j] = v[j];
        }
        seg += (int64_t)v.size();
    }
    return true;
}

}  // namespace

extern "C" {

int64_t rtgpu_gen_blob_words(const rtgpu_gen_params *p) {
    const int n = p->n_tasks, m = p->n_subtasks;
    const int pm = m < 2 ? 0 : (p->mem_model == RTGPU_ONE_COPY ? m - 1 : 2 * m - 2);
    const int64_t seg = (int64_t)n * (2 * m + 2 * pm + 4 * (m - 1));
    return RTGPU_HDR_WORDS + (int64_t)n * RTGPU_REC_WORDS(p->seg_int32) + (p->seg_int32 ? (seg + 1) / 2 : seg);
}

int rtgpu_generate(const rtgpu_gen_params *p, int64_t n_sets, const int64_t *int_seeds,
                   const char *const *str_seeds, int n_threads, int64_t *blobs,
                   int64_t *set_off, int64_t *task_base) {
    if (p->n_tasks < 1 || p->n_subtasks < 1 || p->n_tasks > RTGPU_MAX_TASKS ||
        p->n_subtasks > RTGPU_MAX_M || p->util_num <= 0 || p->util_den <= 0 ||
        p->cpu_lo > p->cpu_hi || p->gpu_lo > p->gpu_hi || p->mem_lo > p->mem_hi ||
        p->cpu_lo < 0 || p->gpu_lo < 0 || p->mem_lo < 0 || p->lofrac_den <= 0 ||
        p->lofrac_num <= 0 || p->lofrac_num > p->lofrac_den || p->eps_den <= 0)
        return -1;
    if (p->seg_int32 && (p->cpu_hi > 0x3fffffff || p->gpu_hi > 0x3fffffff || p->mem_hi > 0x1fffffff))
        return -1; /* segment values (and the merged copies) must fit int32 */
    const int64_t words = rtgpu_gen_blob_words(p);
    for (int64_t s = 0; s <= n_sets; s++) {
        set_off[s] = s * words;
        task_base[s] = s * p->n_tasks;
    }
    if (n_threads < 1) n_threads = 1;
    std::vector<std::thread> th;
    std::vector<char> bad(n_threads, 0);
    for (int t = 0; t < n_threads; t++)
        th.emplace_back([=, &bad]() {
            MT g;
            for (int64_t s = t; s < n_sets; s += n_threads) {
                if (str_seeds) seed_str(g, str_seeds[s]);
                else seed_int(g, int_seeds[s]);
                if (!gen_one(p, g, blobs + s * words)) bad[t] = 1;
            }
        });
    for (auto &x : th) x.join();
    for (char b : bad)
        if (b) return -2; /* a deadline beyond int64 */
    return 0;
}

/* SHA-512 of a buffer (exposed for tests of the seeding path) */
void rtgpu_sha512(const unsigned char *msg, int64_t len, unsigned char *out64) {
    sha512(msg, (size_t)len, out64);
}

}  // extern "C"
