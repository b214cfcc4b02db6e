/*
 * linoct_oracle.c -- CPU restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).
 *
 * See linoct_oracle.h.  Plain C99, scalar, no OpenMP.  Build without -march=native (or
 * with -ffp-contract=off): the reference's FP64 expressions are evaluated without FMA
 * contraction, and so are these.
 */
#include "linoct_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------ */
/* mt19937_64 (the generator rng.hpp builds on; output pinned by the C++ standard).      */

#define MT_N 312
#define MT_M 156

void or_mt_seed(or_mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i) {
        const uint64_t prev = g->mt[i - 1];
        g->mt[i] = 6364136223846793005ULL * (prev ^ (prev >> 62)) + (uint64_t)i;
    }
    g->idx = MT_N;
}

static void mt_refill(or_mt64* g) {
    const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
    for (int i = 0; i < MT_N; ++i) {
        const uint64_t x = (g->mt[i] & upper) | (g->mt[(i + 1) % MT_N] & lower);
        uint64_t xa = x >> 1;
        if (x & 1u) xa ^= 0xB5026F5AA96619E9ULL;
        g->mt[i] = g->mt[(i + MT_M) % MT_N] ^ xa;
    }
    g->idx = 0;
}

uint64_t or_mt_next(or_mt64* g) {
    if (g->idx >= MT_N) mt_refill(g);
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

/* rng.hpp:18-20: 53 random bits scaled to [0,1) */
double or_uniform_double(or_mt64* g) { return (double)(or_mt_next(g) >> 11) * 0x1.0p-53; }

/* rng.hpp:23-32: masked rejection on the bit width of n-1 */
uint64_t or_uniform_below(or_mt64* g, uint64_t n) {
    if (n <= 1) return 0;
    const int bits = 64 - __builtin_clzll(n - 1);
    const uint64_t mask = bits == 64 ? ~0ULL : ((1ULL << bits) - 1);
    uint64_t x;
    do {
        x = or_mt_next(g) & mask;
    } while (x >= n);
    return x;
}

/* rng.hpp:35-42: Box-Muller, u1 redrawn while <= 0 */
double or_gaussian(or_mt64* g) {
    double u1;
    do {
        u1 = or_uniform_double(g);
    } while (u1 <= 0.0);
    const double u2 = or_uniform_double(g);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
}

/* rng.hpp:46-58: partial Fisher-Yates, draw order */
void or_sample_indices(uint32_t n, uint32_t k, uint64_t seed, uint32_t* out) {
    uint32_t* pool = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
    for (uint32_t i = 0; i < n; ++i) pool[i] = i;
    or_mt64 g;
    or_mt_seed(&g, seed);
    const uint32_t take = k < n ? k : n;
    for (uint32_t i = 0; i < take; ++i) {
        const uint32_t j = i + (uint32_t)or_uniform_below(&g, n - i);
        const uint32_t t = pool[i];
        pool[i] = pool[j];
        pool[j] = t;
    }
    memcpy(out, pool, sizeof(uint32_t) * take);
    free(pool);
}

/* ------------------------------------------------------------------------------------ */
/* Synthetic clouds                                                                      */

/* io.cpp:122-130 (gen_uniform): x, y, z each uniform_double * extent, in that order */
void or_gen_uniform(uint64_t n, uint64_t seed, double extent, double* xyz) {
    or_mt64 g;
    or_mt_seed(&g, seed);
    for (uint64_t i = 0; i < n; ++i) {
        xyz[3 * i + 0] = or_uniform_double(&g) * extent;
        xyz[3 * i + 1] = or_uniform_double(&g) * extent;
        xyz[3 * i + 2] = or_uniform_double(&g) * extent;
    }
}

static void terrain_points(or_mt64* g, uint64_t n, double extent_xy, double* xyz) {
    for (uint64_t i = 0; i < n; ++i) {
        const double x = or_uniform_double(g) * extent_xy;
        const double y = or_uniform_double(g) * extent_xy;
        const double s = 10.0 * sin(x / 50.0) * cos(y / 70.0);
        const double z = s + 0.1 * or_gaussian(g);
        xyz[3 * i + 0] = x;
        xyz[3 * i + 1] = y;
        xyz[3 * i + 2] = z;
    }
}

/* cfg1 terrain: x,y = U*extent; z = 10 sin(x/50) cos(y/70) + 0.1 N(0,1) */
void or_gen_terrain(uint64_t n, uint64_t seed, double extent_xy, double* xyz) {
    or_mt64 g;
    or_mt_seed(&g, seed);
    terrain_points(&g, n, extent_xy, xyz);
}

/* cfg3 mixed: 70% terrain over [0,3000)^2, 20% clusters (1000 centres
 * uniform in the terrain bbox, sigma 2), 10% noise with z in [-20,60); one stream. */
void or_gen_mixed(uint64_t n, uint64_t seed, double* xyz) {
    or_mt64 g;
    or_mt_seed(&g, seed);
    const uint64_t nt = n * 7 / 10;
    const uint64_t nc = n * 2 / 10;
    const uint64_t nn = n - nt - nc;
    terrain_points(&g, nt, 3000.0, xyz);
    double box[6];
    if (nt > 0) {
        or_bbox(xyz, nt, box);
    } else {
        for (int a = 0; a < 3; ++a) box[a] = 0.0, box[3 + a] = 3000.0;
    }
    double centres[1000][3];
    for (int c = 0; c < 1000; ++c) {
        for (int a = 0; a < 3; ++a) centres[c][a] = box[a] + or_uniform_double(&g) * (box[3 + a] - box[a]);
    }
    double* p = xyz + 3 * nt;
    for (uint64_t i = 0; i < nc; ++i) {
        const double* c = centres[or_uniform_below(&g, 1000)];
        p[3 * i + 0] = c[0] + 2.0 * or_gaussian(&g);
        p[3 * i + 1] = c[1] + 2.0 * or_gaussian(&g);
        p[3 * i + 2] = c[2] + 2.0 * or_gaussian(&g);
    }
    p += 3 * nc;
    for (uint64_t i = 0; i < nn; ++i) {
        p[3 * i + 0] = or_uniform_double(&g) * 3000.0;
        p[3 * i + 1] = or_uniform_double(&g) * 3000.0;
        p[3 * i + 2] = -20.0 + or_uniform_double(&g) * 80.0;
    }
}

/* ------------------------------------------------------------------------------------ */
/* Geometry + discretizer                                                                */

/* geometry.hpp:64-82: finite check, then running min/max seeded with point 0 */
int64_t or_bbox(const double* xyz, uint64_t n, double box[6]) {
    for (uint64_t i = 0; i < n; ++i) {
        if (!isfinite(xyz[3 * i]) || !isfinite(xyz[3 * i + 1]) || !isfinite(xyz[3 * i + 2]))
            return -1 - (int64_t)i;
    }
    if (n == 0) return 0;
    for (int a = 0; a < 3; ++a) box[a] = box[3 + a] = xyz[a];
    for (uint64_t i = 0; i < n; ++i) {
        for (int a = 0; a < 3; ++a) {
            const double v = xyz[3 * i + a];
            if (v < box[a]) box[a] = v;        /* std::min(cur, v) keeps cur on ties */
            if (box[3 + a] < v) box[3 + a] = v; /* std::max(cur, v) keeps cur on ties */
        }
    }
    return 0;
}

/* geometry.hpp:47-57 */
void or_cubify(const double in[6], double out[6]) {
    double side = in[3] - in[0];
    if (side < in[4] - in[1]) side = in[4] - in[1];
    if (side < in[5] - in[2]) side = in[5] - in[2];
    for (int a = 0; a < 3; ++a) {
        const double m = in[a] + side;
        out[a] = in[a];
        out[3 + a] = m < in[3 + a] ? in[3 + a] : m;
    }
}

/* sfc.cpp:77-80 */
double or_axis_scale(double lo, double hi, int level) {
    const double extent = hi - lo;
    return extent > 0.0 ? ldexp(1.0, level) / extent : 0.0;
}

/* sfc.hpp:104-109 (closed-box check) and :120-124 (floor, clamp to [0, 2^level-1]) */
int or_disc_cell(const double box[6], const double scale[3], int level, const double p[3],
                 uint32_t cell[3]) {
    for (int a = 0; a < 3; ++a) {
        if (!(p[a] >= box[a] && p[a] <= box[3 + a])) return -1;
    }
    const double top = (double)((1ULL << level) - 1);
    for (int a = 0; a < 3; ++a) {
        double u = floor((p[a] - box[a]) * scale[a]);
        if (u < 0.0) u = 0.0;
        else if (top < u) u = top;
        cell[a] = (uint32_t)u;
    }
    return 0;
}

/* sfc.hpp:31-39: bit i of the 21-bit input lands at bit 3i (magic-mask spread) */
uint64_t or_spread3(uint64_t v) {
    v &= 0x1fffffULL;
    v = (v | v << 32) & 0x001f00000000ffffULL;
    v = (v | v << 16) & 0x001f0000ff0000ffULL;
    v = (v | v << 8) & 0x100f00f00f00f00fULL;
    v = (v | v << 4) & 0x10c30c30c30c30c3ULL;
    v = (v | v << 2) & 0x1249249249249249ULL;
    return v;
}

/* sfc.hpp:42-50: inverse of the spread (gathers bits 0,3,6,...) -- written as a loop */
uint32_t or_compact3(uint64_t v) {
    uint32_t out = 0;
    for (int i = 0; i < 21; ++i) out |= (uint32_t)((v >> (3 * i)) & 1u) << i;
    return out;
}

/* sfc.hpp:56-62: x -> MSB of each octal digit, then y, then z */
uint64_t or_morton_encode(uint32_t x, uint32_t y, uint32_t z) {
    return (or_spread3(x) << 2) | (or_spread3(y) << 1) | or_spread3(z);
}

void or_morton_decode(uint64_t code, uint32_t out[3]) {
    out[0] = or_compact3(code >> 2);
    out[1] = or_compact3(code >> 1);
    out[2] = or_compact3(code);
}

/* sfc.cpp:8-42: Skilling's axes-to-transpose Hilbert mapping with the reference's frozen
 * orientation, then the transposed words are interleaved like a Morton code. */
uint64_t or_hilbert_encode(uint32_t x, uint32_t y, uint32_t z, int level) {
    if (level == 0) return 0;
    uint32_t a[3] = {x, y, z};
    const uint32_t top = 1u << (level - 1);
    for (uint32_t q = top; q > 1; q >>= 1) {
        const uint32_t lowmask = q - 1;
        for (int i = 0; i < 3; ++i) {
            if (a[i] & q) {
                a[0] ^= lowmask; /* invert */
            } else {
                const uint32_t sw = (a[0] ^ a[i]) & lowmask; /* exchange low bits */
                a[0] ^= sw;
                a[i] ^= sw;
            }
        }
    }
    a[1] ^= a[0];
    a[2] ^= a[1];
    uint32_t fix = 0;
    for (uint32_t q = top; q > 1; q >>= 1)
        if (a[2] & q) fix ^= q - 1;
    for (int i = 0; i < 3; ++i) a[i] ^= fix;
    return or_morton_encode(a[0], a[1], a[2]);
}

/* sfc.cpp:44-73: transpose-to-axes */
void or_hilbert_decode(uint64_t code, int level, uint32_t out[3]) {
    if (level == 0) {
        out[0] = out[1] = out[2] = 0;
        return;
    }
    const uint32_t mask = (1u << level) - 1;
    uint32_t a[3];
    or_morton_decode(code, a);
    for (int i = 0; i < 3; ++i) a[i] &= mask;
    const uint32_t stop = 2u << (level - 1);
    const uint32_t t = a[2] >> 1;
    a[2] ^= a[1];
    a[1] ^= a[0];
    a[0] ^= t;
    for (uint32_t q = 2; q != stop; q <<= 1) {
        const uint32_t lowmask = q - 1;
        for (int i = 2; i >= 0; --i) {
            if (a[i] & q) {
                a[0] ^= lowmask;
            } else {
                const uint32_t sw = (a[0] ^ a[i]) & lowmask;
                a[0] ^= sw;
                a[i] ^= sw;
            }
        }
    }
    out[0] = a[0];
    out[1] = a[1];
    out[2] = a[2];
}

static void sfc_decode(int curve, uint64_t code, int level, uint32_t out[3]) {
    if (curve == 0) or_morton_decode(code, out);
    else or_hilbert_decode(code, level, out);
}

static uint64_t sfc_encode(int curve, const uint32_t c[3], int level) {
    return curve == 0 ? or_morton_encode(c[0], c[1], c[2]) : or_hilbert_encode(c[0], c[1], c[2], level);
}

/* Signature of a node = the octant digit (x<<2|y<<1|z) of each of its 8 children in code
 * order, read off the decoder one level down (sfc.cpp:145-155). */
static uint32_t child_signature(int curve, uint64_t prefix, int depth) {
    uint32_t sig = 0;
    for (int c = 0; c < 8; ++c) {
        uint32_t cell[3];
        sfc_decode(curve, prefix * 8 + (uint64_t)c, depth + 1, cell);
        sig |= (((cell[0] & 1u) << 2) | ((cell[1] & 1u) << 1) | (cell[2] & 1u)) << (3 * c);
    }
    return sig;
}

/* sfc.cpp:157-194: breadth-first closure of reachable signatures from the root */
int or_stepper(int curve, uint8_t digit[][8], uint8_t next[][8], int max_states) {
    uint32_t sigs[128];
    uint64_t ex_prefix[128];
    int ex_depth[128];
    int count = 0;
    sigs[count] = child_signature(curve, 0, 0);
    ex_prefix[count] = 0;
    ex_depth[count] = 0;
    ++count;
    for (int s = 0; s < count; ++s) {
        if (s >= max_states) return -1;
        for (int c = 0; c < 8; ++c) {
            digit[s][c] = (uint8_t)((sigs[s] >> (3 * c)) & 7u);
            const uint64_t cp = ex_prefix[s] * 8 + (uint64_t)c;
            const uint32_t sig = child_signature(curve, cp, ex_depth[s] + 1);
            int found = -1;
            for (int t = 0; t < count; ++t)
                if (sigs[t] == sig) found = t;
            if (found < 0) {
                if (count >= 128) return -1;
                sigs[count] = sig;
                ex_prefix[count] = cp;
                ex_depth[count] = ex_depth[s] + 1;
                found = count++;
            }
            next[s][c] = (uint8_t)found;
        }
    }
    return count;
}

/* sfc.cpp:84-95: +-2 ulps through the order-preserving integer image of a double */
static uint64_t order_key(double v) {
    uint64_t u;
    memcpy(&u, &v, 8);
    return (u & 0x8000000000000000ULL) ? ~u : (u | 0x8000000000000000ULL);
}
static double from_order_key(uint64_t k) {
    const uint64_t u = (k & 0x8000000000000000ULL) ? (k & 0x7fffffffffffffffULL) : ~k;
    double v;
    memcpy(&v, &u, 8);
    return v;
}

/* sfc.cpp:110-127 */
void or_octant_bounds(const double box[6], uint32_t hx, uint32_t hy, uint32_t hz, int depth,
                      double out[6]) {
    if (depth == 0) {
        memcpy(out, box, sizeof(double) * 6);
        return;
    }
    const double inv = ldexp(1.0, -depth);
    const uint32_t h[3] = {hx, hy, hz};
    for (int a = 0; a < 3; ++a) {
        const double side = (box[3 + a] - box[a]) * inv;
        const double lo = box[a] + (double)h[a] * side;
        const double hi = lo + side;
        out[a] = from_order_key(order_key(lo) - 2);
        out[3 + a] = from_order_key(order_key(hi) + 2);
    }
}

/* ------------------------------------------------------------------------------------ */
/* reorder.cpp                                                                           */

int or_compute_codes(const double* xyz, uint64_t n, int curve, int level, uint64_t* codes,
                     double disc_box[6], double scale[3]) {
    if (n == 0) return -1;
    double box[6], cube[6], sc[3];
    if (or_bbox(xyz, n, box) != 0) return -1;
    or_cubify(box, cube);
    for (int a = 0; a < 3; ++a) sc[a] = or_axis_scale(cube[a], cube[3 + a], level);
    for (uint64_t i = 0; i < n; ++i) {
        uint32_t cell[3];
        if (or_disc_cell(cube, sc, level, xyz + 3 * i, cell) != 0) return -2;
        codes[i] = sfc_encode(curve, cell, level);
    }
    if (disc_box) memcpy(disc_box, cube, sizeof(cube));
    if (scale) memcpy(scale, sc, sizeof(sc));
    return 0;
}

/* Stable order of the codes.  The reference uses an LSD byte radix sort
 * (reorder.cpp:38-62); any stable sort yields the same permutation, here a bottom-up
 * merge sort on (code, original index). */
static void stable_order(const uint64_t* codes, uint64_t n, uint32_t* order) {
    uint32_t* tmp = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
    for (uint64_t i = 0; i < n; ++i) order[i] = (uint32_t)i;
    uint32_t* src = order;
    uint32_t* dst = tmp;
    for (uint64_t w = 1; w < n; w *= 2) {
        for (uint64_t lo = 0; lo < n; lo += 2 * w) {
            const uint64_t mid = lo + w < n ? lo + w : n;
            const uint64_t hi = lo + 2 * w < n ? lo + 2 * w : n;
            uint64_t a = lo, b = mid, o = lo;
            while (a < mid && b < hi) dst[o++] = codes[src[b]] < codes[src[a]] ? src[b++] : src[a++];
            while (a < mid) dst[o++] = src[a++];
            while (b < hi) dst[o++] = src[b++];
        }
        uint32_t* t = src;
        src = dst;
        dst = t;
    }
    if (src != order) memcpy(order, src, sizeof(uint32_t) * n);
    free(tmp);
}

int or_reorder(const double* xyz, uint64_t n, int curve, int level, double* xyz_sorted,
               uint64_t* codes_sorted, uint32_t* perm, double disc_box[6]) {
    if (n == 0 || n > 0xffffffffULL) return -1;
    uint64_t* codes = (uint64_t*)malloc(sizeof(uint64_t) * n);
    const int rc = or_compute_codes(xyz, n, curve, level, codes, disc_box, NULL);
    if (rc != 0) {
        free(codes);
        return rc;
    }
    stable_order(codes, n, perm);
    for (uint64_t i = 0; i < n; ++i) {
        const uint32_t o = perm[i];
        codes_sorted[i] = codes[o];
        if (xyz_sorted) memcpy(xyz_sorted + 3 * i, xyz + 3 * (uint64_t)o, 24);
    }
    free(codes);
    return 0;
}

/* ------------------------------------------------------------------------------------ */
/* linear_octree.cpp                                                                     */

static uint32_t lower_rank(const uint64_t* codes, uint64_t n, uint64_t key) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (codes[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return (uint32_t)lo;
}

/* linear_octree.cpp:23-76: refinement rounds; a block splits into its 8 aligned sub-blocks
 * iff it holds more than n_max points and spans more than one cell. */
int64_t or_build_leaves(const uint64_t* codes, uint64_t n, uint32_t n_max, int level,
                        uint64_t* boundaries, uint32_t* offsets, uint64_t cap) {
    if (n_max < 1 || n == 0) return -1;
    for (uint64_t i = 1; i < n; ++i)
        if (codes[i - 1] > codes[i]) return -1;
    const uint64_t full = 1ULL << (3 * level);
    if (codes[n - 1] >= full) return -1;

    uint64_t m = 1;
    uint64_t* b = (uint64_t*)malloc(sizeof(uint64_t) * 2);
    uint32_t* r = (uint32_t*)malloc(sizeof(uint32_t) * 2);
    b[0] = 0;
    b[1] = full;
    r[0] = 0;
    r[1] = (uint32_t)n;
    for (;;) {
        uint64_t grown = 0;
        for (uint64_t i = 0; i < m; ++i)
            grown += (r[i + 1] - r[i] > n_max && b[i + 1] - b[i] > 1) ? 8 : 1;
        if (grown == m) break;
        uint64_t* nb = (uint64_t*)malloc(sizeof(uint64_t) * (grown + 1));
        uint32_t* nr = (uint32_t*)malloc(sizeof(uint32_t) * (grown + 1));
        uint64_t o = 0;
        for (uint64_t i = 0; i < m; ++i) {
            if (r[i + 1] - r[i] > n_max && b[i + 1] - b[i] > 1) {
                const uint64_t sub = (b[i + 1] - b[i]) >> 3;
                for (int c = 0; c < 8; ++c) nb[o++] = b[i] + (uint64_t)c * sub;
            } else {
                nb[o++] = b[i];
            }
        }
        nb[grown] = full;
        for (uint64_t j = 0; j <= grown; ++j) nr[j] = lower_rank(codes, n, nb[j]);
        free(b);
        free(r);
        b = nb;
        r = nr;
        m = grown;
    }
    int64_t ret = (int64_t)m;
    if (boundaries == NULL) {
        /* size query */
    } else if (m + 1 > cap) {
        ret = -(int64_t)(m + 1) - 2;
    } else {
        memcpy(boundaries, b, sizeof(uint64_t) * (m + 1));
        memcpy(offsets, r, sizeof(uint32_t) * (m + 1));
    }
    free(b);
    free(r);
    return ret;
}

typedef struct {
    const uint64_t* b;
    const uint32_t* off;
    int level;
    or_node* nodes;
    uint64_t cap;
    uint64_t count;
    int bad;
} link_state;

/* linear_octree.cpp:113-137: preorder; a one-leaf range is the leaf itself (~id) */
static int32_t link_range(link_state* st, uint32_t lo, uint32_t hi, uint64_t prefix, int depth) {
    if (hi - lo == 1) return ~(int32_t)lo;
    if (st->count >= st->cap || depth >= st->level) {
        st->bad = 1;
        return 0;
    }
    const uint64_t id = st->count++;
    or_node* nd = &st->nodes[id];
    memset(nd, 0, sizeof(*nd));
    nd->prefix = prefix;
    nd->begin = st->off[lo];
    nd->end = st->off[hi];
    nd->depth = (uint8_t)depth;
    const uint64_t sub = (1ULL << (3 * (st->level - depth))) >> 3;
    uint32_t cursor = lo;
    for (int c = 0; c < 8; ++c) {
        const uint64_t child_end = prefix + (uint64_t)(c + 1) * sub;
        uint32_t nx = cursor;
        while (nx + 1 < hi && st->b[nx + 1] < child_end) ++nx;
        if (st->b[nx + 1] != child_end) {
            st->bad = 1;
            return 0;
        }
        const int32_t child = link_range(st, cursor, nx + 1, prefix + (uint64_t)c * sub, depth + 1);
        if (st->bad) return 0;
        st->nodes[id].children[c] = child;
        uint32_t cb, ce;
        if (child < 0) {
            cb = st->off[~child];
            ce = st->off[~child + 1];
        } else {
            cb = st->nodes[child].begin;
            ce = st->nodes[child].end;
        }
        if (cb != ce) st->nodes[id].child_mask |= (uint8_t)(1u << c);
        cursor = nx + 1;
    }
    return (int32_t)id;
}

int64_t or_link(const uint64_t* boundaries, const uint32_t* offsets, uint64_t leaves, int level,
                or_node* nodes, uint64_t cap, int32_t* root) {
    link_state st = {boundaries, offsets, level, nodes, cap, 0, 0};
    *root = link_range(&st, 0, (uint32_t)leaves, 0, 0);
    if (st.bad) return -1;
    return (int64_t)st.count;
}

/* ------------------------------------------------------------------------------------ */
/* Brute-force search oracles (tests/support/oracles.hpp:19-45) and digests              */

/* geometry.hpp:127-140, strict '<'; shape 0 Sphere, 1 Circle, 2 Cube, 3 Square */
static int contains(int shape, const double c[3], double r, double r2, const double p[3]) {
    const double dx = p[0] - c[0], dy = p[1] - c[1], dz = p[2] - c[2];
    switch (shape) {
        case 0: return dx * dx + dy * dy + dz * dz < r2;
        case 1: return dx * dx + dy * dy < r2;
        case 2: {
            double m = fabs(dx);
            if (m < fabs(dy)) m = fabs(dy);
            if (m < fabs(dz)) m = fabs(dz);
            return m < r;
        }
        default: {
            double m = fabs(dx);
            if (m < fabs(dy)) m = fabs(dy);
            return m < r;
        }
    }
}

uint64_t or_radius_brute(const double* xyz, uint64_t n, const double c[3], double r, int shape,
                         uint32_t* out) {
    const double r2 = r * r; /* geometry.hpp:107, computed once */
    uint64_t k = 0;
    for (uint64_t i = 0; i < n; ++i)
        if (contains(shape, c, r, r2, xyz + 3 * i)) {
            if (out) out[k] = (uint32_t)i;
            ++k;
        }
    return k;
}

typedef struct {
    double d;
    uint32_t i;
} dist_idx;

static int by_dist_then_index(const void* pa, const void* pb) {
    const dist_idx* a = (const dist_idx*)pa;
    const dist_idx* b = (const dist_idx*)pb;
    if (a->d != b->d) return a->d < b->d ? -1 : 1;
    return a->i < b->i ? -1 : (a->i > b->i);
}

/* oracles.hpp:29-45: exact (dist_sq, index) order, k > n returns all n */
uint32_t or_knn_brute(const double* xyz, uint64_t n, const double c[3], uint32_t k, uint32_t* idx,
                      double* dist) {
    dist_idx* all = (dist_idx*)malloc(sizeof(dist_idx) * (n ? n : 1));
    for (uint64_t i = 0; i < n; ++i) {
        const double dx = xyz[3 * i] - c[0], dy = xyz[3 * i + 1] - c[1], dz = xyz[3 * i + 2] - c[2];
        all[i].d = dx * dx + dy * dy + dz * dz;
        all[i].i = (uint32_t)i;
    }
    qsort(all, n, sizeof(dist_idx), by_dist_then_index);
    const uint32_t take = (uint64_t)k < n ? k : (uint32_t)n;
    for (uint32_t j = 0; j < take; ++j) {
        idx[j] = all[j].i;
        if (dist) dist[j] = all[j].d;
    }
    free(all);
    return take;
}

/* search.cpp:263-271: FNV-1a-64 over the 8 little-endian bytes of a value */
uint64_t or_fnv_u64(uint64_t h, uint64_t v) {
    for (int i = 0; i < 8; ++i) {
        h ^= (v >> (8 * i)) & 0xffu;
        h *= 0x100000001b3ULL;
    }
    return h;
}

/* search.cpp:345-347 */
uint64_t or_fnv_radius_row(const uint32_t* idx, uint64_t count) {
    uint64_t h = 0xcbf29ce484222325ULL;
    for (uint64_t j = 0; j < count; ++j) h = or_fnv_u64(h, idx[j]);
    return h;
}

/* search.cpp:376-381: index, then the bit pattern of dist_sq */
uint64_t or_fnv_knn_row(const uint32_t* idx, const double* dist, uint64_t count) {
    uint64_t h = 0xcbf29ce484222325ULL;
    for (uint64_t j = 0; j < count; ++j) {
        uint64_t bits;
        memcpy(&bits, &dist[j], 8);
        h = or_fnv_u64(h, idx[j]);
        h = or_fnv_u64(h, bits);
    }
    return h;
}

/* ------------------------------------------------------------------------------------ */
/* neighbours_struct (search.cpp:76-135): pruned traversal over the octant boxes          */

/* kernel_octant_relation (geometry.hpp:197-231): 0 Contains, 1 Disjoint, 2 Intersects */
static int octant_relation(int shape, const double c[3], double r, double r2, const double b[6]) {
    double nr[3], fr[3];
    for (int a = 0; a < 3; ++a) {
        double nn = b[a] - c[a];
        if (c[a] - b[3 + a] > nn) nn = c[a] - b[3 + a];
        if (0.0 > nn) nn = 0.0;
        const double f1 = c[a] - b[a], f2 = b[3 + a] - c[a];
        nr[a] = nn;
        fr[a] = f1 < f2 ? f2 : f1;  /* std::max(a, b) returns a unless a < b */
    }
    double nm, fm, lim;
    switch (shape) {
        case 0:
            nm = nr[0] * nr[0] + nr[1] * nr[1] + nr[2] * nr[2];
            fm = fr[0] * fr[0] + fr[1] * fr[1] + fr[2] * fr[2];
            lim = r2;
            break;
        case 1:
            nm = nr[0] * nr[0] + nr[1] * nr[1];
            fm = fr[0] * fr[0] + fr[1] * fr[1];
            lim = r2;
            break;
        case 2:
            nm = nr[0]; if (nm < nr[1]) nm = nr[1]; if (nm < nr[2]) nm = nr[2];
            fm = fr[0]; if (fm < fr[1]) fm = fr[1]; if (fm < fr[2]) fm = fr[2];
            lim = r;
            break;
        default:
            nm = nr[0]; if (nm < nr[1]) nm = nr[1];
            fm = fr[0]; if (fm < fr[1]) fm = fr[1];
            lim = r;
            break;
    }
    if (fm < lim) return 0;
    if (nm >= lim) return 1;
    return 2;
}

int64_t or_radius_struct(const double* xyz, const uint64_t* boundaries, const uint32_t* offsets,
                         const or_node* nodes, int32_t root, const double disc_box[6], int level,
                         int curve, const double c[3], double r, int shape, uint32_t* ranges,
                         uint64_t cap_ranges, uint32_t* singles, uint64_t cap_singles,
                         uint64_t* n_ranges, uint64_t* n_singles) {
    const double r2 = r * r;
    uint64_t nr = 0, ns = 0, count = 0;
    int32_t stack[8 * 64 + 8];
    int sp = 0;
    stack[sp++] = root;  /* reorder rejects empty clouds, so the tree has points */
    while (sp > 0) {
        const int32_t ref = stack[--sp];
        uint64_t prefix;
        int depth;
        uint32_t b, e;
        if (ref < 0) {
            const uint32_t id = (uint32_t)~ref;
            prefix = boundaries[id];
            const uint64_t span = boundaries[id + 1] - boundaries[id];
            int lg = 0;
            while ((1ULL << (3 * lg)) < span) ++lg;
            depth = level - lg;
            b = offsets[id];
            e = offsets[id + 1];
        } else {
            prefix = nodes[ref].prefix;
            depth = nodes[ref].depth;
            b = nodes[ref].begin;
            e = nodes[ref].end;
        }
        /* prefix_to_octant_bounds (sfc.cpp:129-141) == the Frame's CurveStepper coordinates */
        uint32_t cell[3];
        sfc_decode(curve, prefix, level, cell);
        const int sh = level - depth;
        double box[6];
        or_octant_bounds(disc_box, sh >= 32 ? 0 : cell[0] >> sh, sh >= 32 ? 0 : cell[1] >> sh,
                         sh >= 32 ? 0 : cell[2] >> sh, depth, box);
        const int rel = octant_relation(shape, c, r, r2, box);
        if (rel == 1) continue;
        if (rel == 0) {  /* search.cpp:124-129: adjacent ranges coalesce */
            if (nr > 0 && ranges[2 * (nr - 1) + 1] == b) {
                ranges[2 * (nr - 1) + 1] = e;
            } else {
                if (nr >= cap_ranges) return -1;
                ranges[2 * nr] = b;
                ranges[2 * nr + 1] = e;
                ++nr;
            }
            count += e - b;
            continue;
        }
        if (ref < 0) {
            for (uint32_t i = b; i < e; ++i)
                if (contains(shape, c, r, r2, xyz + 3 * (uint64_t)i)) {
                    if (ns >= cap_singles) return -1;
                    singles[ns++] = i;
                    ++count;
                }
        } else {
            for (int ch = 7; ch >= 0; --ch) {  /* push_children (search.cpp:30-41) */
                const int32_t cr = nodes[ref].children[ch];
                uint32_t cb, ce;
                if (cr < 0) {
                    cb = offsets[~cr];
                    ce = offsets[~cr + 1];
                } else {
                    cb = nodes[cr].begin;
                    ce = nodes[cr].end;
                }
                if (cb == ce) continue;
                if (sp >= (int)(sizeof stack / sizeof stack[0])) return -1;
                stack[sp++] = cr;
            }
        }
    }
    *n_ranges = nr;
    *n_singles = ns;
    return (int64_t)count;
}

/* search.cpp:325-336: ranges as (begin << 32 | end), a separator, then the singles */
uint64_t or_fnv_struct_row(const uint32_t* ranges, uint64_t n_ranges, const uint32_t* singles,
                           uint64_t n_singles) {
    uint64_t h = 0xcbf29ce484222325ULL;
    for (uint64_t j = 0; j < n_ranges; ++j)
        h = or_fnv_u64(h, ((uint64_t)ranges[2 * j] << 32) | ranges[2 * j + 1]);
    h = or_fnv_u64(h, 0xffffffffffffffffULL);
    for (uint64_t j = 0; j < n_singles; ++j) h = or_fnv_u64(h, singles[j]);
    return h;
}
