/*
 * linoct_oracle.h -- CPU restatement of the reference hot path (TEST INFRASTRUCTURE).
 *
 * This is the parity oracle, not product code.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it, and only as the checker.  The product path
 * (paper_2603_06771_b200) never links or calls anything here.
 *
 * Pinned against: the reference's own known-answer tests (tests/golden/kat.json, from
 * proj/tests/test_sfc.cpp:62-125, test_linear_octree.cpp:26-34) and golden vectors produced
 * by the reference library itself compiled from /root/reference (oracle/_ref, see
 * tests/golden/make_golden.py).
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj).
 */
#ifndef LINOCT_ORACLE_H
#define LINOCT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng.hpp:1-60 ---------------------------------------------------------------- */
typedef struct {
    uint64_t mt[312];
    int idx;
} or_mt64;

void or_mt_seed(or_mt64* g, uint64_t seed);
uint64_t or_mt_next(or_mt64* g);
double or_uniform_double(or_mt64* g);                 /* rng.hpp:18-20 */
uint64_t or_uniform_below(or_mt64* g, uint64_t n);   /* rng.hpp:23-32 */
double or_gaussian(or_mt64* g);                       /* rng.hpp:35-42 */
void or_sample_indices(uint32_t n, uint32_t k, uint64_t seed, uint32_t* out); /* rng.hpp:46-58 */

/* ---- generators (io.cpp:122-130; terrain / mixed per SURVEY.md §8d) --------------- */
void or_gen_uniform(uint64_t n, uint64_t seed, double extent, double* xyz);
void or_gen_terrain(uint64_t n, uint64_t seed, double extent_xy, double* xyz);
void or_gen_mixed(uint64_t n, uint64_t seed, double* xyz);

/* ---- geometry.hpp / sfc ------------------------------------------------------------ */
/* bbox of AoS xyz (geometry.hpp:64-82); returns -1 - index of first non-finite point,
 * 0 on success.  box = {minx,miny,minz,maxx,maxy,maxz}. */
int64_t or_bbox(const double* xyz, uint64_t n, double box[6]);
void or_cubify(const double in[6], double out[6]);              /* geometry.hpp:47-57 */
double or_axis_scale(double lo, double hi, int level);          /* sfc.cpp:77-80 */
/* cell of one point (sfc.hpp:104-109, :120-124); returns 0, or -1 when outside the box */
int or_disc_cell(const double box[6], const double scale[3], int level, const double p[3],
                 uint32_t cell[3]);
uint64_t or_spread3(uint64_t v);                                /* sfc.hpp:31-39 */
uint32_t or_compact3(uint64_t v);                               /* sfc.hpp:42-50 */
uint64_t or_morton_encode(uint32_t x, uint32_t y, uint32_t z);  /* sfc.hpp:56-62 */
void or_morton_decode(uint64_t code, uint32_t out[3]);          /* sfc.hpp:64-68 */
uint64_t or_hilbert_encode(uint32_t x, uint32_t y, uint32_t z, int level); /* sfc.cpp:8-42 */
void or_hilbert_decode(uint64_t code, int level, uint32_t out[3]);          /* sfc.cpp:44-73 */
/* CurveStepper closure (sfc.cpp:143-237): writes digit[s][c], next[s][c]; returns #states */
int or_stepper(int curve, uint8_t digit[][8], uint8_t next[][8], int max_states);
/* octant_bounds with the 2-ulp pads (sfc.cpp:84-95, :110-127) */
void or_octant_bounds(const double box[6], uint32_t hx, uint32_t hy, uint32_t hz, int depth,
                      double out[6]);

/* ---- reorder.cpp ------------------------------------------------------------------- */
/* compute_codes (reorder.cpp:9-26) on the cubified bbox; disc_box/scale out optional */
int or_compute_codes(const double* xyz, uint64_t n, int curve, int level, uint64_t* codes,
                     double disc_box[6], double scale[3]);
/* reorder_cloud (reorder.cpp:66-89): stable sort by code, AoS gather */
int or_reorder(const double* xyz, uint64_t n, int curve, int level, double* xyz_sorted,
               uint64_t* codes_sorted, uint32_t* perm, double disc_box[6]);

/* ---- linear_octree.cpp ------------------------------------------------------------- */
/* build_leaves (linear_octree.cpp:23-76).  Returns leaf count L (boundaries has L+1
 * entries), or -1 on invalid input, or -(needed) - 2 when cap is too small. */
int64_t or_build_leaves(const uint64_t* codes, uint64_t n, uint32_t n_max, int level,
                        uint64_t* boundaries, uint32_t* offsets, uint64_t cap);

/* InternalNode, layout identical to linear_octree.hpp:46-53 (56 bytes) */
typedef struct {
    uint64_t prefix;
    int32_t children[8];
    uint32_t begin;
    uint32_t end;
    uint8_t depth;
    uint8_t child_mask;
    uint8_t pad_[6];
} or_node;

/* link_internal / link_range (linear_octree.cpp:107-137).  Returns internal count and
 * writes *root; nodes must hold >= L/7 + 8 entries. */
int64_t or_link(const uint64_t* boundaries, const uint32_t* offsets, uint64_t leaves,
                int level, or_node* nodes, uint64_t cap, int32_t* root);

/* ---- search (oracles.hpp:19-45 brute-force restatements; search.cpp:263-271 FNV) --- */
uint64_t or_radius_brute(const double* xyz, uint64_t n, const double c[3], double r,
                         int shape, uint32_t* out);
uint32_t or_knn_brute(const double* xyz, uint64_t n, const double c[3], uint32_t k,
                      uint32_t* idx, double* dist);
uint64_t or_fnv_u64(uint64_t h, uint64_t v);
uint64_t or_fnv_radius_row(const uint32_t* idx, uint64_t count);
uint64_t or_fnv_knn_row(const uint32_t* idx, const double* dist, uint64_t count);
/* neighbours_struct (search.cpp:76-135) for one centre over the tree arrays: ranges as
 * (begin, end) pairs, coalesced when adjacent; singles ascending.  Returns the member
 * count (RangedResult::count), or -1 when a capacity is exceeded. */
int64_t or_radius_struct(const double* xyz, const uint64_t* boundaries, const uint32_t* offsets,
                         const or_node* nodes, int32_t root, const double disc_box[6], int level,
                         int curve, const double c[3], double r, int shape, uint32_t* ranges,
                         uint64_t cap_ranges, uint32_t* singles, uint64_t cap_singles,
                         uint64_t* n_ranges, uint64_t* n_singles);
/* search.cpp:325-336: the Struct row digest */
uint64_t or_fnv_struct_row(const uint32_t* ranges, uint64_t n_ranges, const uint32_t* singles,
                           uint64_t n_singles);

#ifdef __cplusplus
}
#endif
#endif
