/*
 * spc_oracle.c -- plain, slow, obviously-correct CPU oracle for the Spira SpC hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see spc_oracle.h).  Nothing here is shared with, or
 * reachable from, the CUDA product path.  Each function cites the passage of
 * /root/reference/PAPER.md (P:line) it writes out.
 *
 * Build: gcc -O2 -std=c11 -fPIC -shared spc_oracle.c -o liboracle.so
 */
#include "spc_oracle.h"

#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------
 * canonical order (§5.2 "lexicographically sorted")
 * ---------------------------------------------------------------------------------- */

typedef struct {
    int32_t c[4];
    int32_t row;
} orc_row;

static int cmp_tuple(const int32_t *a, const int32_t *b) {
    for (int d = 0; d < 4; ++d) {
        if (a[d] < b[d]) return -1;
        if (a[d] > b[d]) return 1;
    }
    return 0;
}

static int cmp_row(const void *pa, const void *pb) {
    const orc_row *a = (const orc_row *)pa, *b = (const orc_row *)pb;
    int c = cmp_tuple(a->c, b->c);
    if (c) return c;
    return (a->row > b->row) - (a->row < b->row); /* stable */
}

int64_t orc_sort_coords(const int32_t *coords, int64_t n, int32_t *sorted_out, int32_t *perm_out) {
    if (n < 0) return -1;
    orc_row *r = (orc_row *)malloc(sizeof(orc_row) * (size_t)(n ? n : 1));
    if (!r) return -1;
    for (int64_t i = 0; i < n; ++i) {
        memcpy(r[i].c, coords + 4 * i, 16);
        r[i].row = (int32_t)i;
    }
    qsort(r, (size_t)n, sizeof(orc_row), cmp_row);
    int64_t dups = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (sorted_out) memcpy(sorted_out + 4 * i, r[i].c, 16);
        if (perm_out) perm_out[i] = r[i].row;
        if (i > 0 && cmp_tuple(r[i - 1].c, r[i].c) == 0) ++dups;
    }
    free(r);
    return dups;
}

/* ------------------------------------------------------------------------------------
 * packed key (§5.3: x in the most significant bits, then y, then z; the
 * batch field above x and the 2^(b-1) bias per field are DESIGN.md readings A3/A5)
 * ---------------------------------------------------------------------------------- */

int64_t orc_pack(const int32_t *coords, int64_t n, int bits_b, int bits_x, int bits_y, int bits_z,
                 uint64_t *keys_out) {
    int64_t bad = 0;
    const int bits[4] = {bits_b, bits_x, bits_y, bits_z};
    for (int64_t i = 0; i < n; ++i) {
        uint64_t key = 0;
        int ok = 1;
        for (int d = 0; d < 4; ++d) {
            int64_t v = coords[4 * i + d];
            int64_t field = (d == 0) ? v : v + ((int64_t)1 << (bits[d] - 1));
            if (field < 0 || field >= ((int64_t)1 << bits[d])) ok = 0;
            key = (key << bits[d]) | (uint64_t)field;   /* b first => b ends up highest */
        }
        if (!ok) { key = 0; ++bad; }
        keys_out[i] = key;
    }
    return bad;
}

/* ------------------------------------------------------------------------------------
 * Eq. (1) downsampling (§2.1), floor toward -infinity
 * ---------------------------------------------------------------------------------- */

int32_t orc_round_down(int32_t v, int32_t s) {
    int32_t q = v / s;                  /* C division truncates toward zero */
    if ((v % s != 0) && (v < 0)) q -= 1; /* ... so step down for negative non-multiples */
    return q * s;
}

int64_t orc_downsample(const int32_t *coords, int64_t n, int32_t s, int32_t *out) {
    if (s <= 0) return -1;
    int32_t *tmp = (int32_t *)malloc(16 * (size_t)(n ? n : 1));
    if (!tmp) return -1;
    for (int64_t i = 0; i < n; ++i) {
        tmp[4 * i + 0] = coords[4 * i + 0];
        for (int d = 1; d < 4; ++d) tmp[4 * i + d] = orc_round_down(coords[4 * i + d], s);
    }
    int32_t *sorted = (int32_t *)malloc(16 * (size_t)(n ? n : 1));
    if (!sorted) { free(tmp); return -1; }
    orc_sort_coords(tmp, n, sorted, NULL);
    int64_t m = 0;
    for (int64_t i = 0; i < n; ++i) {       /* keep only the unique values */
        if (i > 0 && cmp_tuple(sorted + 4 * (i - 1), sorted + 4 * i) == 0) continue;
        memcpy(out + 4 * m, sorted + 4 * i, 16);
        ++m;
    }
    free(tmp);
    free(sorted);
    return m;
}

/* ------------------------------------------------------------------------------------
 * Delta(K, s_p) (§2.1) in the order of P:266 (group 0 = (-1,-1,-1),(-1,-1,0),(-1,-1,1))
 * ---------------------------------------------------------------------------------- */

int orc_offsets(int K, int spacing, int32_t *off_out, int32_t *l1_units_out) {
    if (K <= 0 || (K % 2) == 0) return -1;
    int r = (K - 1) / 2, k = 0;
    for (int ex = -r; ex <= r; ++ex)
        for (int ey = -r; ey <= r; ++ey)
            for (int ez = -r; ez <= r; ++ez, ++k) {
                if (off_out) {
                    off_out[3 * k + 0] = ex * spacing;
                    off_out[3 * k + 1] = ey * spacing;
                    off_out[3 * k + 2] = ez * spacing;
                }
                if (l1_units_out) l1_units_out[k] = abs(ex) + abs(ey) + abs(ez);
            }
    return k;
}

/* Generalised offset box: per axis K_a offsets; odd K_a centred as in
 * Delta(K, s_p), even K_a = {0, .., K_a - 1} (reading E1: the K = 2 down/up
 * layers' {0, s_p}^3); lexicographic (dx, dy, dz), dz fastest. */
int orc_offsets3(int kx, int ky, int kz, int spacing, int32_t *off_out, int32_t *l1_units_out) {
    if (kx <= 0 || ky <= 0 || kz <= 0) return -1;
    const int lx = (kx % 2) ? -(kx - 1) / 2 : 0, ly = (ky % 2) ? -(ky - 1) / 2 : 0, lz = (kz % 2) ? -(kz - 1) / 2 : 0;
    int k = 0;
    for (int ex = lx; ex < lx + kx; ++ex)
        for (int ey = ly; ey < ly + ky; ++ey)
            for (int ez = lz; ez < lz + kz; ++ez, ++k) {
                if (off_out) {
                    off_out[3 * k + 0] = ex * spacing;
                    off_out[3 * k + 1] = ey * spacing;
                    off_out[3 * k + 2] = ez * spacing;
                }
                if (l1_units_out) l1_units_out[k] = abs(ex) + abs(ey) + abs(ez);
            }
    return k;
}

/* ------------------------------------------------------------------------------------
 * hash set over (b,x,y,z) tuples -> canonical index (open addressing, linear probing)
 * ---------------------------------------------------------------------------------- */

typedef struct {
    const int32_t *coords;
    int64_t *slot; /* index+1, 0 = empty */
    uint64_t mask;
} orc_hash;

static uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

static uint64_t hash_tuple(const int32_t *t) {
    uint64_t h = 0x9e3779b97f4a7c15ULL;
    for (int d = 0; d < 4; ++d) h = mix64(h ^ (uint64_t)(uint32_t)t[d]);
    return h;
}

static int hash_build(orc_hash *h, const int32_t *coords, int64_t n) {
    uint64_t cap = 16;
    while (cap < (uint64_t)(2 * n + 1)) cap <<= 1;
    h->slot = (int64_t *)calloc(cap, sizeof(int64_t));
    if (!h->slot) return -1;
    h->mask = cap - 1;
    h->coords = coords;
    for (int64_t i = 0; i < n; ++i) {
        uint64_t p = hash_tuple(coords + 4 * i) & h->mask;
        while (h->slot[p]) p = (p + 1) & h->mask;
        h->slot[p] = i + 1;
    }
    return 0;
}

static int64_t hash_find(const orc_hash *h, const int32_t *t) {
    uint64_t p = hash_tuple(t) & h->mask;
    while (h->slot[p]) {
        int64_t j = h->slot[p] - 1;
        if (cmp_tuple(h->coords + 4 * j, t) == 0) return j;
        p = (p + 1) & h->mask;
    }
    return -1;
}

/* the query of Eq. (2)'s indicator: p = q + delta_k (normal) or p = q - delta_k (transposed) */
static void make_query(const int32_t *q, const int32_t *off, int transposed, int32_t *t) {
    t[0] = q[0];
    for (int d = 0; d < 3; ++d) t[d + 1] = transposed ? q[d + 1] - off[d] : q[d + 1] + off[d];
}

/* ------------------------------------------------------------------------------------
 * kernel map (§2.2): M[i,k] = j if q_i + delta_k matches p_j, else -1
 * ---------------------------------------------------------------------------------- */

static int64_t kmap_impl(const int32_t *in_coords, int64_t n_in, const int32_t *out_coords, int64_t n_out,
                         const int32_t *off, int kv, int transposed, int32_t *triples, int64_t cap) {
    orc_hash h;
    if (hash_build(&h, in_coords, n_in)) return -1;
    int64_t nnz = 0;
    int32_t t[4];
    for (int k = 0; k < kv; ++k)
        for (int64_t i = 0; i < n_out; ++i) {
            make_query(out_coords + 4 * i, off + 3 * k, transposed, t);
            int64_t j = hash_find(&h, t);
            if (j < 0) continue;
            if (triples && nnz < cap) {
                triples[3 * nnz + 0] = k;
                triples[3 * nnz + 1] = (int32_t)i;
                triples[3 * nnz + 2] = (int32_t)j;
            }
            ++nnz;
        }
    free(h.slot);
    return nnz;
}

/* the offset table of Delta(K, s_p) (cubic odd K) or of the generalised box */
static int32_t *offset_table(int kx, int ky, int kz, int cubic_odd_only, int spacing, int *kv) {
    *kv = cubic_odd_only ? orc_offsets(kx, 1, NULL, NULL) : orc_offsets3(kx, ky, kz, 1, NULL, NULL);
    if (*kv < 0) return NULL;
    int32_t *off = (int32_t *)malloc(sizeof(int32_t) * 3 * (size_t)*kv);
    if (cubic_odd_only) orc_offsets(kx, spacing, off, NULL);
    else orc_offsets3(kx, ky, kz, spacing, off, NULL);
    return off;
}

int64_t orc_kmap(const int32_t *in_coords, int64_t n_in, const int32_t *out_coords, int64_t n_out,
                 int K, int spacing, int transposed, int32_t *triples, int64_t cap) {
    int kv;
    int32_t *off = offset_table(K, K, K, 1, spacing, &kv);
    if (!off) return -1;
    int64_t r = kmap_impl(in_coords, n_in, out_coords, n_out, off, kv, transposed, triples, cap);
    free(off);
    return r;
}

int64_t orc_kmap3(const int32_t *in_coords, int64_t n_in, const int32_t *out_coords, int64_t n_out,
                  int kx, int ky, int kz, int spacing, int transposed, int32_t *triples, int64_t cap) {
    int kv;
    int32_t *off = offset_table(kx, ky, kz, 0, spacing, &kv);
    if (!off) return -1;
    int64_t r = kmap_impl(in_coords, n_in, out_coords, n_out, off, kv, transposed, triples, cap);
    free(off);
    return r;
}

/* ------------------------------------------------------------------------------------
 * Eq. (2) in fp64 (§2.1), two loop orders (§2.2 dataflows)
 * ---------------------------------------------------------------------------------- */

static void axpy_row(const double *f, int c_in, const double *Wk, int c_out, double *acc) {
    for (int ci = 0; ci < c_in; ++ci) {
        double a = f[ci];
        const double *w = Wk + (size_t)ci * c_out;
        for (int co = 0; co < c_out; ++co) acc[co] += a * w[co];
    }
}

static int64_t conv_impl(const int32_t *in_coords, int64_t n_in, const int32_t *out_coords, int64_t n_out,
                         const int32_t *off, int kv, int transposed, const double *F_in, int c_in,
                         const double *W, int c_out, double *F_out, int order) {
    if (c_in <= 0 || c_out <= 0) return -1;
    orc_hash h;
    if (hash_build(&h, in_coords, n_in)) return -1;
    memset(F_out, 0, sizeof(double) * (size_t)n_out * (size_t)c_out);
    int64_t nnz = 0;
    int32_t t[4];
    if (order == 0) { /* output-stationary: each output row finished before the next */
        /* rows are independent (each row's sum runs in the same order either way): the
         * OpenMP build (liboracle_omp.so) spreads them over the host cores */
#pragma omp parallel for reduction(+ : nnz) schedule(dynamic, 64)
        for (int64_t i = 0; i < n_out; ++i)
            for (int k = 0; k < kv; ++k) {
                int32_t t[4];
                make_query(out_coords + 4 * i, off + 3 * k, transposed, t);
                int64_t j = hash_find(&h, t);
                if (j < 0) continue;
                axpy_row(F_in + (size_t)j * c_in, c_in, W + (size_t)k * c_in * c_out, c_out,
                         F_out + (size_t)i * c_out);
                ++nnz;
            }
    } else {          /* weight-stationary: one offset at a time, partial sums merged */
        for (int k = 0; k < kv; ++k)
            for (int64_t i = 0; i < n_out; ++i) {
                make_query(out_coords + 4 * i, off + 3 * k, transposed, t);
                int64_t j = hash_find(&h, t);
                if (j < 0) continue;
                axpy_row(F_in + (size_t)j * c_in, c_in, W + (size_t)k * c_in * c_out, c_out,
                         F_out + (size_t)i * c_out);
                ++nnz;
            }
    }
    free(h.slot);
    return nnz;
}

int64_t orc_conv(const int32_t *in_coords, int64_t n_in, const int32_t *out_coords, int64_t n_out,
                 int K, int spacing, int transposed, const double *F_in, int c_in,
                 const double *W, int c_out, double *F_out, int order) {
    int kv;
    int32_t *off = offset_table(K, K, K, 1, spacing, &kv);
    if (!off) return -1;
    int64_t r = conv_impl(in_coords, n_in, out_coords, n_out, off, kv, transposed, F_in, c_in, W, c_out, F_out, order);
    free(off);
    return r;
}

int64_t orc_conv3(const int32_t *in_coords, int64_t n_in, const int32_t *out_coords, int64_t n_out,
                  int kx, int ky, int kz, int spacing, int transposed, const double *F_in, int c_in,
                  const double *W, int c_out, double *F_out, int order) {
    int kv;
    int32_t *off = offset_table(kx, ky, kz, 0, spacing, &kv);
    if (!off) return -1;
    int64_t r = conv_impl(in_coords, n_in, out_coords, n_out, off, kv, transposed, F_in, c_in, W, c_out, F_out, order);
    free(off);
    return r;
}

static int64_t conv_rows_impl(const int32_t *in_coords, int64_t n_in, const int32_t *out_coords,
                              const int64_t *rows, int64_t n_rows, const int32_t *off, int kv, int transposed,
                              const double *F_in, int c_in, const double *W, int c_out, double *F_out) {
    orc_hash h;
    if (hash_build(&h, in_coords, n_in)) return -1;
    memset(F_out, 0, sizeof(double) * (size_t)n_rows * (size_t)c_out);
    int64_t nnz = 0;
#pragma omp parallel for reduction(+ : nnz) schedule(dynamic, 64)
    for (int64_t r = 0; r < n_rows; ++r)
        for (int k = 0; k < kv; ++k) {
            int32_t t[4];
            make_query(out_coords + 4 * rows[r], off + 3 * k, transposed, t);
            int64_t j = hash_find(&h, t);
            if (j < 0) continue;
            axpy_row(F_in + (size_t)j * c_in, c_in, W + (size_t)k * c_in * c_out, c_out,
                     F_out + (size_t)r * c_out);
            ++nnz;
        }
    free(h.slot);
    return nnz;
}

int64_t orc_conv_rows(const int32_t *in_coords, int64_t n_in, const int32_t *out_coords,
                      const int64_t *rows, int64_t n_rows, int K, int spacing, int transposed,
                      const double *F_in, int c_in, const double *W, int c_out, double *F_out) {
    int kv;
    int32_t *off = offset_table(K, K, K, 1, spacing, &kv);
    if (!off) return -1;
    int64_t r = conv_rows_impl(in_coords, n_in, out_coords, rows, n_rows, off, kv, transposed, F_in, c_in, W, c_out,
                               F_out);
    free(off);
    return r;
}

int64_t orc_conv_rows3(const int32_t *in_coords, int64_t n_in, const int32_t *out_coords,
                       const int64_t *rows, int64_t n_rows, int kx, int ky, int kz, int spacing, int transposed,
                       const double *F_in, int c_in, const double *W, int c_out, double *F_out) {
    int kv;
    int32_t *off = offset_table(kx, ky, kz, 0, spacing, &kv);
    if (!off) return -1;
    int64_t r = conv_rows_impl(in_coords, n_in, out_coords, rows, n_rows, off, kv, transposed, F_in, c_in, W, c_out,
                               F_out);
    free(off);
    return r;
}

/* ------------------------------------------------------------------------------------
 * NEXT-4 training path: gradients of Eq. (2) (§2.1; training is beyond the
 * paper's scope).  Same matches as conv_impl; the gradient of f_out_i w.r.t. f_j is
 * W_k^T and w.r.t. W_k is f_j^T (x) d f_out_i.
 * ---------------------------------------------------------------------------------- */

int64_t orc_conv_dgrad3(const int32_t *in_coords, int64_t n_in, const int32_t *out_coords, int64_t n_out,
                        int kx, int ky, int kz, int spacing, int transposed, const double *dF_out, int c_out,
                        const double *W, int c_in, double *dF_in) {
    int kv;
    int32_t *off = offset_table(kx, ky, kz, 0, spacing, &kv);
    if (!off || c_in <= 0 || c_out <= 0) { free(off); return -1; }
    orc_hash h;
    if (hash_build(&h, in_coords, n_in)) { free(off); return -1; }
    memset(dF_in, 0, sizeof(double) * (size_t)n_in * (size_t)c_in);
    int64_t nnz = 0;
    for (int64_t i = 0; i < n_out; ++i)
        for (int k = 0; k < kv; ++k) {
            int32_t t[4];
            make_query(out_coords + 4 * i, off + 3 * k, transposed, t);
            int64_t j = hash_find(&h, t);
            if (j < 0) continue;
            const double *g = dF_out + (size_t)i * c_out;
            const double *Wk = W + (size_t)k * c_in * c_out;
            double *d = dF_in + (size_t)j * c_in;
            for (int ci = 0; ci < c_in; ++ci) {
                double s = 0.0;
                for (int co = 0; co < c_out; ++co) s += g[co] * Wk[(size_t)ci * c_out + co];
                d[ci] += s;
            }
            ++nnz;
        }
    free(h.slot);
    free(off);
    return nnz;
}

int64_t orc_conv_dgrad_rows3(const int32_t *in_coords, int64_t n_in, const int32_t *out_coords, int64_t n_out,
                             const int64_t *rows, int64_t n_rows, int kx, int ky, int kz, int spacing,
                             int transposed, const double *dF_out, int c_out, const double *W, int c_in,
                             double *dF_in_rows) {
    (void)n_in;
    int kv;
    int32_t *off = offset_table(kx, ky, kz, 0, spacing, &kv);
    if (!off || c_in <= 0 || c_out <= 0) { free(off); return -1; }
    orc_hash h;   /* hash on the OUTPUT set: which outputs reach input row j */
    if (hash_build(&h, out_coords, n_out)) { free(off); return -1; }
    memset(dF_in_rows, 0, sizeof(double) * (size_t)n_rows * (size_t)c_in);
    int64_t nnz = 0;
#pragma omp parallel for reduction(+ : nnz) schedule(dynamic, 64)
    for (int64_t r = 0; r < n_rows; ++r)
        for (int k = 0; k < kv; ++k) {
            /* p_j = q_i + delta_k  <=>  q_i = p_j - delta_k (transposed: p_j = q_i - delta_k) */
            int32_t t[4];
            make_query(in_coords + 4 * rows[r], off + 3 * k, !transposed, t);
            int64_t i = hash_find(&h, t);
            if (i < 0) continue;
            const double *g = dF_out + (size_t)i * c_out;
            const double *Wk = W + (size_t)k * c_in * c_out;
            double *d = dF_in_rows + (size_t)r * c_in;
            for (int ci = 0; ci < c_in; ++ci) {
                double s = 0.0;
                for (int co = 0; co < c_out; ++co) s += g[co] * Wk[(size_t)ci * c_out + co];
                d[ci] += s;
            }
            ++nnz;
        }
    free(h.slot);
    free(off);
    return nnz;
}

int64_t orc_conv_wgrad3(const int32_t *in_coords, int64_t n_in, const int32_t *out_coords, int64_t n_out,
                        int kx, int ky, int kz, int spacing, int transposed, const double *F_in, int c_in,
                        const double *dF_out, int c_out, double *dW) {
    int kv;
    int32_t *off = offset_table(kx, ky, kz, 0, spacing, &kv);
    if (!off || c_in <= 0 || c_out <= 0) { free(off); return -1; }
    orc_hash h;
    if (hash_build(&h, in_coords, n_in)) { free(off); return -1; }
    memset(dW, 0, sizeof(double) * (size_t)kv * (size_t)c_in * (size_t)c_out);
    int64_t nnz = 0;
    /* one offset at a time: dW_k is a sum over that offset's matches only */
#pragma omp parallel for reduction(+ : nnz) schedule(dynamic, 1)
    for (int k = 0; k < kv; ++k)
        for (int64_t i = 0; i < n_out; ++i) {
            int32_t t[4];
            make_query(out_coords + 4 * i, off + 3 * k, transposed, t);
            int64_t j = hash_find(&h, t);
            if (j < 0) continue;
            const double *f = F_in + (size_t)j * c_in;
            const double *g = dF_out + (size_t)i * c_out;
            double *Wk = dW + (size_t)k * c_in * c_out;
            for (int ci = 0; ci < c_in; ++ci)
                for (int co = 0; co < c_out; ++co) Wk[(size_t)ci * c_out + co] += f[ci] * g[co];
            ++nnz;
        }
    free(h.slot);
    free(off);
    return nnz;
}

void orc_bn_relu(const double *x, int64_t n, int c, const double *gamma, const double *beta, const double *mean,
                 const double *var, double eps, const double *residual, int relu, double *y) {
    for (int64_t i = 0; i < n; ++i)
        for (int ch = 0; ch < c; ++ch) {
            double v = x[(size_t)i * c + ch];
            if (gamma) v = (v - mean[ch]) / sqrt(var[ch] + eps) * gamma[ch] + beta[ch];
            if (residual) v += residual[(size_t)i * c + ch];
            if (relu && v < 0.0) v = 0.0;
            y[(size_t)i * c + ch] = v;
        }
}

/* spconv's "regular" output rule (P:476-478 networks' public definitions):
 * V_out = { (b, p - delta) : p in V_in, delta in the offset box (spacing), every spatial
 * coordinate of p - delta a multiple of out_stride } -- every output site of stride
 * out_stride whose kernel footprint touches an input.  Written sorted and unique to out
 * (room for n * K_x K_y K_z rows).  Returns |V_out| or -1. */
int64_t orc_regular_outputs(const int32_t *in_coords, int64_t n, int kx, int ky, int kz, int spacing,
                            int out_stride, int32_t *out) {
    int kv;
    int32_t *off = offset_table(kx, ky, kz, 0, spacing, &kv);
    if (!off || out_stride < 1) { free(off); return -1; }
    int32_t *cand = (int32_t *)malloc(sizeof(int32_t) * 4 * (size_t)(n * kv > 0 ? n * kv : 1));
    int64_t m = 0;
    for (int64_t i = 0; i < n; ++i)
        for (int k = 0; k < kv; ++k) {
            int32_t c[4] = {in_coords[4 * i], 0, 0, 0};
            int on = 1;
            for (int d = 0; d < 3; ++d) {
                c[1 + d] = in_coords[4 * i + 1 + d] - off[3 * k + d];
                on &= orc_round_down(c[1 + d], out_stride) == c[1 + d];
            }
            if (on) { memcpy(cand + 4 * m, c, sizeof(c)); ++m; }
        }
    int64_t u = orc_downsample(cand, m, 1, out);   /* stride 1: sort + unique */
    free(cand);
    free(off);
    return u;
}

/* ------------------------------------------------------------------------------------
 * voxelization: §2.1 "v_i = floor(p_i^(raw) / g)"; S:70-78 quantize
 * (floor toward -infinity, duplicates merged, point -> voxel index map); S:132 merged
 * voxels' features averaged
 * ---------------------------------------------------------------------------------- */
#include <math.h>

int64_t orc_voxelize(const float *pts, int64_t ld, const int32_t *batch, int64_t n, const float *g,
                     const float *feats, int64_t ld_f, int c, int32_t *coords_out, int32_t *point_voxel,
                     double *feats_out) {
    if (n < 0) return -1;
    orc_row *r = (orc_row *)malloc(sizeof(orc_row) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) {
        r[i].c[0] = batch ? batch[i] : 0;
        for (int d = 0; d < 3; ++d) {
            float p = pts[i * ld + d];
            float q = p / g[d]; /* float32 quotient, IEEE round-to-nearest (reading V1) */
            if (!isfinite(p) || !isfinite(q)) { free(r); return -(1 + i); }
            double v = floor((double)q); /* floor toward -infinity ("floor(-0.6) = -1") */
            if (v < -2147483648.0 || v > 2147483647.0) { free(r); return -(1 + i); }
            r[i].c[1 + d] = (int32_t)v;
        }
        r[i].row = (int32_t)i;
    }
    /* canonical order of the (b, v) rows; equal rows keep ascending point index */
    qsort(r, (size_t)n, sizeof(orc_row), cmp_row);
    int64_t nv = 0;
    if (feats_out) memset(feats_out, 0, sizeof(double) * (size_t)n * (size_t)(c > 0 ? c : 0));
    int64_t first = 0; /* sorted position of the current voxel's first point */
    for (int64_t i = 0; i < n; ++i) {
        if (i == 0 || cmp_tuple(r[i - 1].c, r[i].c) != 0) {
            memcpy(coords_out + 4 * nv, r[i].c, sizeof(int32_t) * 4);
            ++nv;
            first = i;
        }
        const int64_t v = nv - 1;
        if (point_voxel) point_voxel[r[i].row] = (int32_t)v;
        if (feats && feats_out) {
            for (int ch = 0; ch < c; ++ch) feats_out[v * c + ch] += (double)feats[(int64_t)r[i].row * ld_f + ch];
            const int last = (i + 1 == n) || cmp_tuple(r[i].c, r[i + 1].c) != 0;
            if (last)
                for (int ch = 0; ch < c; ++ch) feats_out[v * c + ch] /= (double)(i - first + 1);
        }
    }
    free(r);
    return nv;
}

#ifdef _OPENMP
#include <omp.h>
int orc_num_threads(void) { return omp_get_max_threads(); }
#else
int orc_num_threads(void) { return 1; }
#endif
