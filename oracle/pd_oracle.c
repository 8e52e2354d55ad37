/*
 * pd_oracle.c — CPU restatement of the reference Gray-code Pauli decomposition.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library, and only as the
 * checker or the timed CPU baseline. The product path (paper_2401_16378_b200)
 * never links or calls it and fails loudly when its CUDA extension is missing.
 *
 * Parity pin: tests/test_oracle.py checks every function here against the
 * reference's own known-answer tests (proj/tests/test_decompose.cpp:69-86,
 * proj/tests/python/test_smoke.py:57-65), against golden vectors produced by
 * the reference itself (tests/golden/, made by tests/golden/make_golden.py from
 * the reference pybind module built here), and bit-for-bit against
 * oracle/_ref/libpdref.so (the reference's own sources compiled by
 * oracle/Makefile) on seeded inputs.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * the reference's proj/ directory).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define PDO_EXPORT __attribute__((visibility("default")))

/* bits.hpp:52-55 base4_digit */
static inline unsigned digit(uint64_t n, unsigned t) { return (unsigned)((n >> (2 * t)) & 3u); }

/* pauli.hpp:23-39 is_antidiagonal / xy_mask: bit t set iff digit t is X or Y */
PDO_EXPORT uint64_t pdo_xy_mask(uint64_t n, unsigned num_qubits) {
    uint64_t mask = 0;
    for (unsigned t = 0; t < num_qubits; ++t) {
        unsigned d = digit(n, t);
        mask |= (uint64_t)((d ^ (d >> 1)) & 1u) << t;
    }
    return mask;
}

/* pauli.hpp:54-63 beta_exponent(op, 0) = {0,0,3,0}; pauli.hpp:97-102
 * initial_column_phase = Σ_t beta_exponent(d_t, 0) mod 4 = 3·#Y mod 4 */
PDO_EXPORT unsigned pdo_initial_phase(uint64_t n, unsigned num_qubits) {
    unsigned p = 0;
    for (unsigned t = 0; t < num_qubits; ++t)
        p += digit(n, t) == 2 ? 3u : 0u;
    return p & 3u;
}

/* bits.hpp:37-44 gray_code, flipped_bit_index */
PDO_EXPORT uint64_t pdo_gray_code(uint64_t k) { return k ^ (k >> 1); }
PDO_EXPORT unsigned pdo_flipped_bit_index(uint64_t k) { return (unsigned)__builtin_ctzll(k + 1); }

/*
 * The reference's term is lambda.value() * a[...] (decompose.cpp:40): a
 * std::complex<double> product, which GCC evaluates as (ac - bd, ad + bc) and,
 * when both parts are NaN, passes to libgcc's __muldc3 — the infinity recovery
 * of C99 Annex G.5.1, restated here. lambda = unit_phase(p) (pauli.hpp:71-76).
 */
static void cmul_annex_g(double a, double b, double c, double d, double* re, double* im) {
    const double ac = a * c, bd = b * d, ad = a * d, bc = b * c;
    double x = ac - bd, y = ad + bc;
    if (isnan(x) && isnan(y)) {
        int recalc = 0;
        if (isinf(a) || isinf(b)) { /* first factor infinite: box it, the other's NaNs -> 0 */
            a = copysign(isinf(a) ? 1.0 : 0.0, a);
            b = copysign(isinf(b) ? 1.0 : 0.0, b);
            if (isnan(c)) c = copysign(0.0, c);
            if (isnan(d)) d = copysign(0.0, d);
            recalc = 1;
        }
        if (isinf(c) || isinf(d)) { /* second factor infinite */
            c = copysign(isinf(c) ? 1.0 : 0.0, c);
            d = copysign(isinf(d) ? 1.0 : 0.0, d);
            if (isnan(a)) a = copysign(0.0, a);
            if (isnan(b)) b = copysign(0.0, b);
            recalc = 1;
        }
        if (!recalc && (isinf(ac) || isinf(bd) || isinf(ad) || isinf(bc))) { /* overflow */
            if (isnan(a)) a = copysign(0.0, a);
            if (isnan(b)) b = copysign(0.0, b);
            if (isnan(c)) c = copysign(0.0, c);
            if (isnan(d)) d = copysign(0.0, d);
            recalc = 1;
        }
        if (recalc) {
            x = INFINITY * (a * c - b * d);
            y = INFINITY * (a * d + b * c);
        }
    }
    *re = x;
    *im = y;
}

static const double kUnitRe[4] = {1.0, 0.0, -1.0, 0.0}; /* pauli.hpp:71-76 unit_phase */
static const double kUnitIm[4] = {0.0, 1.0, 0.0, -1.0};

/* acc += i^lam · (er + i ei). For a finite element the product is the exact re/im swap with
 * sign (the reference's product up to the sign of an exact zero); an infinite or NaN element
 * takes the reference's full complex product, whose 0·inf terms are NaN. */
static inline void add_term(unsigned lam, double er, double ei, double* ar, double* ai) {
    if (!(isfinite(er) && isfinite(ei))) {
        double tr, ti;
        cmul_annex_g(kUnitRe[lam], kUnitIm[lam], er, ei, &tr, &ti);
        *ar += tr;
        *ai += ti;
        return;
    }
    switch (lam) { /* i^lam · (er + i ei) */
        case 0: *ar += er; *ai += ei; break;
        case 1: *ar += -ei; *ai += er; break;
        case 2: *ar += -er; *ai += -ei; break;
        default: *ar += ei; *ai += -er; break;
    }
}

/*
 * decompose.cpp:30-47 gray_walk_sum + :49-57 coeff_fast_impl.
 * λ is a 2-bit power of i (pauli.hpp:91-125); λ·a is add_term above. The walk visits
 * i = gray(k) for k = 0..dim-1 and after each step multiplies λ by the row-flip
 * quotient of the digit at the flipped bit: -1 for Y and Z (pauli.hpp:66-68).
 */
static void coeff_fast_raw(unsigned N, const double* g, uint64_t n, double* out) {
    const uint64_t dim = (uint64_t)1 << N;
    const uint64_t mask = pdo_xy_mask(n, N);
    unsigned lam = pdo_initial_phase(n, N);
    double ar = 0.0, ai = 0.0;
    uint64_t code = 0;
    for (uint64_t step = 0;; ++step) {
        const double* e = g + 2 * ((code ^ mask) * dim + code);
        add_term(lam, e[0], e[1], &ar, &ai);
        if (step + 1 == dim) break;
        const unsigned t = (unsigned)__builtin_ctzll(step + 1);
        lam = (lam + ((digit(n, t) >> 1) ? 2u : 0u)) & 3u;
        code ^= (uint64_t)1 << t;
    }
    out[0] = ar / (double)dim; /* decompose.cpp:56: exact division by 2^N */
    out[1] = ai / (double)dim;
}

/* decompose.cpp:14-19 check_index, bits.hpp:63-65 valid_pauli_index */
static int bad_index(unsigned N, uint64_t n) { return N < 32 && n >= ((uint64_t)1 << (2 * N)); }

PDO_EXPORT int pdo_coeff_fast(unsigned N, const double* g, uint64_t n, double* out) {
    if (N == 0 || N > 31 || bad_index(N, n)) return -1;
    coeff_fast_raw(N, g, n, out);
    return 0;
}

/* decompose.cpp:59-80 coeff_slow_impl: λ rebuilt per step from the N-factor
 * product of beta(op_t, bit_t(i)) (pauli.hpp:54-63). */
PDO_EXPORT int pdo_coeff_slow(unsigned N, const double* g, uint64_t n, double* out) {
    static const unsigned beta[4][2] = {{0, 0}, {0, 0}, {3, 1}, {0, 2}};
    if (N == 0 || N > 31 || bad_index(N, n)) return -1;
    const uint64_t dim = (uint64_t)1 << N;
    const uint64_t mask = pdo_xy_mask(n, N);
    double ar = 0.0, ai = 0.0;
    for (uint64_t k = 0; k < dim; ++k) {
        const uint64_t i = k ^ (k >> 1);
        unsigned lam = 0;
        for (unsigned t = 0; t < N; ++t) lam += beta[digit(n, t)][(i >> t) & 1u];
        const double* e = g + 2 * ((i ^ mask) * dim + i);
        add_term(lam & 3u, e[0], e[1], &ar, &ai);
    }
    out[0] = ar / (double)dim;
    out[1] = ai / (double)dim;
    return 0;
}

typedef struct {
    unsigned N;
    const double* g;
    const uint64_t* ns; /* NULL => n = begin..end */
    uint64_t begin, end;
    double* out;
} job_t;

static void* run_job(void* arg) {
    job_t* j = (job_t*)arg;
    for (uint64_t k = j->begin; k < j->end; ++k) {
        const uint64_t n = j->ns ? j->ns[k] : k;
        coeff_fast_raw(j->N, j->g, n, j->out + 2 * k);
    }
    return NULL;
}

/* decompose.cpp:95-131 decompose_parallel_impl: contiguous static split of
 * the index range over threads; here generalised to an explicit index list. */
static int run_split(unsigned N, const double* g, const uint64_t* ns, uint64_t total, double* out,
                     unsigned threads) {
    if (threads == 0) return -1;
    const uint64_t chunk = total == 0 ? 1 : (total + threads - 1) / threads;
    unsigned used = (unsigned)(total == 0 ? 0 : (total + chunk - 1) / chunk);
    if (used <= 1) {
        job_t j = {N, g, ns, 0, total, out};
        run_job(&j);
        return 0;
    }
    pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * used);
    job_t* jobs = (job_t*)malloc(sizeof(job_t) * used);
    for (unsigned w = 0; w < used; ++w) {
        uint64_t b = (uint64_t)w * chunk, e = b + chunk < total ? b + chunk : total;
        job_t j = {N, g, ns, b, e, out};
        jobs[w] = j;
        pthread_create(&tid[w], NULL, run_job, &jobs[w]);
    }
    for (unsigned w = 0; w < used; ++w) pthread_join(tid[w], NULL);
    free(tid);
    free(jobs);
    return 0;
}

PDO_EXPORT int pdo_decompose(unsigned N, const double* g, double* out, unsigned threads) {
    if (N == 0 || N > 15) return -1;
    return run_split(N, g, NULL, (uint64_t)1 << (2 * N), out, threads);
}

PDO_EXPORT int pdo_coeff_batch(unsigned N, const double* g, const uint64_t* ns, uint64_t count,
                               double* out, unsigned threads) {
    if (N == 0 || N > 31) return -1;
    for (uint64_t k = 0; k < count; ++k)
        if (bad_index(N, ns[k])) return -1;
    return run_split(N, g, ns, count, out, threads);
}

/* decompose.cpp:221-250 recompose: the walk in reverse, row r holds λ_r c_n
 * at column r^mask; exactly-zero coefficients are skipped. */
PDO_EXPORT int pdo_recompose(unsigned N, const double* coeffs, double* out) {
    if (N == 0 || N > 15) return -1;
    const uint64_t dim = (uint64_t)1 << N, total = dim * dim;
    memset(out, 0, sizeof(double) * 2 * total);
    for (uint64_t n = 0; n < total; ++n) {
        const double cr = coeffs[2 * n], ci = coeffs[2 * n + 1];
        if (cr == 0.0 && ci == 0.0) continue;
        const uint64_t mask = pdo_xy_mask(n, N);
        unsigned lam = pdo_initial_phase(n, N);
        uint64_t code = 0;
        for (uint64_t step = 0;; ++step) {
            double* a = out + 2 * (code * dim + (code ^ mask));
            add_term(lam, cr, ci, &a[0], &a[1]);
            if (step + 1 == dim) break;
            const unsigned t = (unsigned)__builtin_ctzll(step + 1);
            lam = (lam + ((digit(n, t) >> 1) ? 2u : 0u)) & 3u;
            code ^= (uint64_t)1 << t;
        }
    }
    return 0;
}

/* bench.cpp:16-22 splitmix64 */
static inline uint64_t splitmix64(uint64_t* state) {
    *state += 0x9E3779B97F4A7C15ull;
    uint64_t z = *state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* bench.cpp:25-27 unit_interval: top 53 bits -> [0,1) -> [-1,1), exact */
static inline double unit_interval(uint64_t bits) {
    return (double)(bits >> 11) * 0x1.0p-53 * 2.0 - 1.0;
}

/* bench.cpp:42-46 matrix_seed */
PDO_EXPORT uint64_t pdo_matrix_seed(uint64_t seed, unsigned num_qubits, unsigned rep) {
    uint64_t state = seed ^ ((uint64_t)num_qubits * 0xD6E8FEB86659FD93ull) ^
                     ((uint64_t)rep * 0xCA5A826395121157ull);
    return splitmix64(&state);
}

/* bench.cpp:48-58 random_matrix: element k takes two draws, re then im */
PDO_EXPORT int pdo_random_matrix(unsigned N, uint64_t seed, double* out) {
    if (N == 0 || N > 15) return -1;
    const uint64_t count = (uint64_t)1 << (2 * N);
    uint64_t state = seed;
    for (uint64_t k = 0; k < count; ++k) {
        out[2 * k] = unit_interval(splitmix64(&state));
        out[2 * k + 1] = unit_interval(splitmix64(&state));
    }
    return 0;
}
