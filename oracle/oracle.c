/*
 * oracle.c — plain, slow, obviously-correct CPU oracle for the Flowtree hot path
 *            (arXiv 1910.04126, "Scalable Nearest Neighbor Search for Optimal Transport").
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path may link, import or execute this
 * file.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs use it (through oracle/__init__.py).  It shares no code, header, table or constant
 * generator with paper_1910_04126_b200/csrc/.
 *
 * Compiled with:  gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -shared -fPIC
 * All floating point is IEEE binary64, round-to-nearest-even, evaluated in exactly the order
 * written (no FMA contraction).
 *
 * Step numbering O1..O10 follows SURVEY.md §8(c); every step cites the PAPER.md passage it
 * follows (PAPER.md line numbers, /root/reference/PAPER.md).
 *
 *   O1  ground normalisation ............ PAPER.md:113 (§2 footnote, coordinates in [0,Φ])
 *   O2  random shift σ .................. PAPER.md:116-117 (§2 "Generic Quadtree")
 *   O3  cell rule ....................... PAPER.md:116-121 (§2, H = [-Φ,Φ]^d + σ, halving)
 *   O4  tree ............................ PAPER.md:121 (§2, non-empty cells, singleton leaves)
 *   O5  node ids, levels, edge weights .. PAPER.md:121-122 (§2, root level log Φ + 1, 2^ℓ)
 *   O6  masses (exact cross-scaling) .... PAPER.md:20-26 (Eq. (1)), :267 (normalised masses)
 *   O7  Quadtree value .................. PAPER.md:126-129 (§2 "Wasserstein-1 on Quadtree")
 *   O8  Flowtree flow ................... PAPER.md:495-504 (App. A.1 "Flowtree Computation")
 *   O9  Flowtree value .................. PAPER.md:141-150 (§3, W~1 = Σ f(x,x')·||x-x'||)
 *   O10 k-NN / prefetch-and-prune ........ PAPER.md:45-49 (§1), :402-431 (§4.4), :987 (Table 7)
 *
 * Readings of the paper where it is silent or garbled are listed in DESIGN.md §3 and are
 * referenced below as "reading R#".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EINVAL 1
#define OR_ERANGE 2
#define OR_EOVERFLOW 3
#define OR_ENOMEM 4
#define OR_ECAP 5

/* ------------------------------------------------------------------------------------------ */
/* O2: SplitMix64 output i for state `seed`, as a pure function of (seed, i) (reading R3).     */
/* ------------------------------------------------------------------------------------------ */
uint64_t or_splitmix64(uint64_t seed, uint64_t i) {
    uint64_t z = seed + (i + 1u) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z = z ^ (z >> 31);
    return z;
}

/* r_i = (z_i >> 11) * 2^-53, uniform in [0,1); σ_i = Φ * r_i. */
void or_sigma_from_seed(uint64_t seed, int32_t d, double phi, double* sigma) {
    for (int32_t i = 0; i < d; i++) {
        uint64_t z = or_splitmix64(seed, (uint64_t)i);
        double r = (double)(z >> 11) * 0x1.0p-53;
        sigma[i] = phi * r;
    }
}

/* ------------------------------------------------------------------------------------------ */
/* Tree                                                                                        */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
    int64_t N;
    int32_t d;
    int32_t D;        /* depth cap: number of halvings allowed */
    int32_t d_star;   /* realised maximum leaf depth */
    int32_t l_root;   /* level of the root, ceil(log2 Φ) + 1 */
    double phi;
    double* mn;       /* [d] per-axis minimum */
    double* sigma;    /* [d] */
    int64_t M;        /* number of nodes */
    int32_t* node_depth;  /* [M] */
    int32_t* node_parent; /* [M], -1 for the root */
    int32_t* node_count;  /* [M] number of ground points in the cell */
    int32_t* leaf_depth;  /* [N] depth of the leaf holding point x */
    int32_t* path;        /* [N * (d_star+1)] node at depth k of point x, -1 below its leaf */
} or_tree;

/* O3: q_{x,i} = min(floor(u * 2^D), 2^D - 1), u = (t + a) / (2Φ), t = x_i - mn_i, a = Φ - σ_i.
 * The depth-k cell coordinate is q >> (D - k).                                               */
static int64_t cell_q(const or_tree* T, const float* X, int64_t x, int32_t i) {
    double t = (double)X[x * T->d + i] - T->mn[i];
    double a = T->phi - T->sigma[i];
    double num = t + a;
    double u = num / (2.0 * T->phi);
    double s = ldexp(u, T->D);
    double f = floor(s);
    int64_t q = (int64_t)f;
    int64_t top = ((int64_t)1 << T->D) - 1;
    if (q > top) q = top;
    return q;
}

/* bit-vector of a point at depth k: bit_i = c^{(k)}_i & 1, compared lexicographically with
 * dimension 0 first (reading R7).  Stored as an array of d bytes for plain comparison.      */
typedef struct {
    int64_t x;
    int64_t d;
    unsigned char* bits;
} bv_item;

static int cmp_bv(const void* pa, const void* pb) {
    const bv_item* a = (const bv_item*)pa;
    const bv_item* b = (const bv_item*)pb;
    int c = memcmp(a->bits, b->bits, (size_t)a->d);
    if (c != 0) return c;
    return (a->x < b->x) ? -1 : (a->x > b->x);
}

void or_tree_free(or_tree* T) {
    if (!T) return;
    free(T->mn); free(T->sigma); free(T->node_depth); free(T->node_parent);
    free(T->node_count); free(T->leaf_depth); free(T->path);
    free(T);
}

/* Build the quadtree over X[N x d] (fp32, row-major).  sigma != NULL gives σ explicitly
 * (test hook); otherwise σ comes from `seed` via O2.  D = depth cap (<= 0 means 32).       */
int or_build(const float* X, int64_t N, int32_t d, const double* sigma, uint64_t seed, int32_t D,
             or_tree** out) {
    *out = NULL;
    if (N < 1 || d < 1) return OR_EINVAL;
    if (D <= 0) D = 32;
    if (D > 52) return OR_EINVAL;
    or_tree* T = (or_tree*)calloc(1, sizeof(or_tree));
    if (!T) return OR_ENOMEM;
    T->N = N; T->d = d; T->D = D;
    T->mn = (double*)malloc(sizeof(double) * (size_t)d);
    T->sigma = (double*)malloc(sizeof(double) * (size_t)d);
    T->leaf_depth = (int32_t*)malloc(sizeof(int32_t) * (size_t)N);

    /* O1: per-axis minimum anchor, Φ = max range. */
    double phi = 0.0;
    for (int32_t i = 0; i < d; i++) {
        double mn = (double)X[i], mx = (double)X[i];
        for (int64_t x = 1; x < N; x++) {
            double v = (double)X[x * d + i];
            if (v < mn) mn = v;
            if (v > mx) mx = v;
        }
        T->mn[i] = mn;
        double r = mx - mn;
        if (r > phi) phi = r;
    }
    T->phi = phi;

    /* O2 */
    if (sigma) { for (int32_t i = 0; i < d; i++) T->sigma[i] = sigma[i]; }
    else or_sigma_from_seed(seed, d, phi, T->sigma);

    /* O5: root level ceil(log2 Φ) + 1 computed exactly with frexp. */
    if (phi > 0.0) {
        int e; double m = frexp(phi, &e);     /* phi = m * 2^e, m in [0.5, 1) */
        int cl = (m == 0.5) ? (e - 1) : e;    /* ceil(log2 phi) */
        T->l_root = cl + 1;
    } else {
        T->l_root = 0;
    }

    /* O4 / O5: breadth-first construction.  Node arrays grow as needed. */
    int64_t cap = 1024, M = 1;
    int32_t* nd = (int32_t*)malloc(sizeof(int32_t) * (size_t)cap);
    int32_t* np = (int32_t*)malloc(sizeof(int32_t) * (size_t)cap);
    int32_t* nc = (int32_t*)malloc(sizeof(int32_t) * (size_t)cap);
    /* members: points of each node at the current frontier, stored as one array ordered by node */
    int64_t* cur_pts = (int64_t*)malloc(sizeof(int64_t) * (size_t)N);
    int64_t* nxt_pts = (int64_t*)malloc(sizeof(int64_t) * (size_t)N);
    int64_t* cur_start = NULL; int64_t* cur_len = NULL; int64_t* cur_node = NULL; int64_t n_cur = 0;
    /* history of node-at-depth per point: per depth an array [N] (−1 if not present) */
    int32_t** at_depth = (int32_t**)calloc((size_t)D + 1, sizeof(int32_t*));
    if (!nd || !np || !nc || !cur_pts || !nxt_pts || !at_depth) { or_tree_free(T); return OR_ENOMEM; }

    nd[0] = 0; np[0] = -1; nc[0] = (int32_t)N;
    at_depth[0] = (int32_t*)malloc(sizeof(int32_t) * (size_t)N);
    for (int64_t x = 0; x < N; x++) { at_depth[0][x] = 0; cur_pts[x] = x; T->leaf_depth[x] = 0; }
    int32_t d_star = 0;

    /* the root splits iff it holds >= 2 points, Φ > 0 and the cap allows a halving */
    int root_internal = (N >= 2 && phi > 0.0 && D >= 1);
    if (root_internal) {
        n_cur = 1;
        cur_start = (int64_t*)malloc(sizeof(int64_t)); cur_len = (int64_t*)malloc(sizeof(int64_t));
        cur_node = (int64_t*)malloc(sizeof(int64_t));
        cur_start[0] = 0; cur_len[0] = N; cur_node[0] = 0;
    }
    unsigned char* bitbuf = (unsigned char*)malloc((size_t)N * (size_t)d);
    bv_item* items = (bv_item*)malloc(sizeof(bv_item) * (size_t)N);

    for (int32_t k = 1; k <= D && n_cur > 0; k++) {
        at_depth[k] = (int32_t*)malloc(sizeof(int32_t) * (size_t)N);
        for (int64_t x = 0; x < N; x++) at_depth[k][x] = -1;
        int64_t* nxt_start = (int64_t*)malloc(sizeof(int64_t) * (size_t)N);
        int64_t* nxt_len = (int64_t*)malloc(sizeof(int64_t) * (size_t)N);
        int64_t* nxt_node = (int64_t*)malloc(sizeof(int64_t) * (size_t)N);
        int64_t n_nxt = 0, fill = 0;
        /* parents in ID order (the frontier is kept in node-ID order) */
        for (int64_t p = 0; p < n_cur; p++) {
            int64_t st = cur_start[p], len = cur_len[p];
            for (int64_t j = 0; j < len; j++) {
                int64_t x = cur_pts[st + j];
                unsigned char* b = bitbuf + (size_t)(st + j) * (size_t)d;
                for (int32_t i = 0; i < d; i++) {
                    int64_t q = cell_q(T, X, x, i);
                    int64_t c = q >> (D - k);       /* depth-k cell coordinate */
                    b[i] = (unsigned char)(c & 1);
                }
                items[j].x = x; items[j].d = d; items[j].bits = b;
            }
            qsort(items, (size_t)len, sizeof(bv_item), cmp_bv);
            /* group equal bit-vectors into children, in bit-vector order */
            int64_t j = 0;
            while (j < len) {
                int64_t e = j + 1;
                while (e < len && memcmp(items[e].bits, items[j].bits, (size_t)d) == 0) e++;
                if (M == cap) {
                    cap *= 2;
                    nd = (int32_t*)realloc(nd, sizeof(int32_t) * (size_t)cap);
                    np = (int32_t*)realloc(np, sizeof(int32_t) * (size_t)cap);
                    nc = (int32_t*)realloc(nc, sizeof(int32_t) * (size_t)cap);
                }
                int64_t v = M++;
                nd[v] = k; np[v] = (int32_t)cur_node[p]; nc[v] = (int32_t)(e - j);
                for (int64_t t = j; t < e; t++) {
                    at_depth[k][items[t].x] = (int32_t)v;
                    T->leaf_depth[items[t].x] = k;
                }
                if (k > d_star) d_star = k;
                /* a child with >= 2 points below the cap splits further; else it is a leaf */
                if ((e - j) >= 2 && k < D) {
                    nxt_start[n_nxt] = fill; nxt_len[n_nxt] = e - j; nxt_node[n_nxt] = v; n_nxt++;
                    for (int64_t t = j; t < e; t++) nxt_pts[fill++] = items[t].x;
                }
                j = e;
            }
        }
        free(cur_start); free(cur_len); free(cur_node);
        cur_start = nxt_start; cur_len = nxt_len; cur_node = nxt_node; n_cur = n_nxt;
        int64_t* tmp = cur_pts; cur_pts = nxt_pts; nxt_pts = tmp;
    }
    free(cur_start); free(cur_len); free(cur_node);
    free(bitbuf); free(items); free(cur_pts); free(nxt_pts);

    T->M = M; T->node_depth = nd; T->node_parent = np; T->node_count = nc; T->d_star = d_star;
    T->path = (int32_t*)malloc(sizeof(int32_t) * (size_t)N * (size_t)(d_star + 1));
    for (int64_t x = 0; x < N; x++)
        for (int32_t k = 0; k <= d_star; k++)
            T->path[x * (d_star + 1) + k] = (k <= D && at_depth[k]) ? at_depth[k][x] : -1;
    for (int32_t k = 0; k <= D; k++) free(at_depth[k]);
    free(at_depth);
    *out = T;
    return OR_OK;
}

void or_tree_info(const or_tree* T, double* phi, int32_t* l_root, int32_t* d_star, int64_t* n_nodes) {
    if (phi) *phi = T->phi;
    if (l_root) *l_root = T->l_root;
    if (d_star) *d_star = T->d_star;
    if (n_nodes) *n_nodes = T->M;
}
void or_tree_vectors(const or_tree* T, double* mn, double* sigma) {
    for (int32_t i = 0; i < T->d; i++) { if (mn) mn[i] = T->mn[i]; if (sigma) sigma[i] = T->sigma[i]; }
}
void or_tree_paths(const or_tree* T, int32_t* out) {
    memcpy(out, T->path, sizeof(int32_t) * (size_t)T->N * (size_t)(T->d_star + 1));
}
void or_tree_nodes(const or_tree* T, int32_t* depth, int32_t* parent, int32_t* count) {
    for (int64_t v = 0; v < T->M; v++) {
        if (depth) depth[v] = T->node_depth[v];
        if (parent) parent[v] = T->node_parent[v];
        if (count) count[v] = T->node_count[v];
    }
}

/* ------------------------------------------------------------------------------------------ */
/* Distributions                                                                               */
/* ------------------------------------------------------------------------------------------ */
typedef struct { int32_t id; uint32_t w; } or_entry;
static int cmp_entry(const void* a, const void* b) {
    int32_t x = ((const or_entry*)a)->id, y = ((const or_entry*)b)->id;
    return (x < y) ? -1 : (x > y);
}

/* copies a support into an id-sorted array, validating it (reading R17: reject zero masses and
 * duplicate ids; ids must be in [0, N)).                                                     */
static int load_support(const or_tree* T, const int32_t* ids, const uint32_t* w, int32_t s,
                        or_entry** out, uint64_t* total) {
    if (s < 1) return OR_EINVAL;
    or_entry* e = (or_entry*)malloc(sizeof(or_entry) * (size_t)s);
    uint64_t tot = 0;
    for (int32_t i = 0; i < s; i++) {
        if (ids[i] < 0 || (int64_t)ids[i] >= T->N) { free(e); return OR_ERANGE; }
        if (w[i] == 0) { free(e); return OR_EINVAL; }
        e[i].id = ids[i]; e[i].w = w[i]; tot += w[i];
    }
    qsort(e, (size_t)s, sizeof(or_entry), cmp_entry);
    for (int32_t i = 1; i < s; i++) if (e[i].id == e[i - 1].id) { free(e); return OR_EINVAL; }
    if (tot > 65535u) { free(e); return OR_EOVERFLOW; }   /* W, U <= 65535 keeps W*U < 2^32 */
    *out = e; *total = tot;
    return OR_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* O6 + O7: Quadtree closed form  Σ_{v != root} 2^{ℓ(v)} |μ(v) − ν(v)|        */
/* ------------------------------------------------------------------------------------------ */
typedef struct { int32_t node; uint64_t m; } nm_pair;
static int cmp_nm(const void* a, const void* b) {
    int32_t x = ((const nm_pair*)a)->node, y = ((const nm_pair*)b)->node;
    return (x < y) ? -1 : (x > y);
}

/* node masses as (node, subtree sum) for non-root nodes, sorted by node id.  Masses are the
 * cross-scaled integers μ'(x) = w_x * other_total.                                          */
static int64_t node_masses(const or_tree* T, const or_entry* e, int32_t s, uint64_t scale, nm_pair** out) {
    int32_t h = T->d_star + 1;
    nm_pair* raw = (nm_pair*)malloc(sizeof(nm_pair) * ((size_t)s * (size_t)h + 1));
    int64_t n = 0;
    for (int32_t i = 0; i < s; i++) {
        int32_t x = e[i].id;
        for (int32_t k = 1; k <= T->leaf_depth[x]; k++) {
            raw[n].node = T->path[(int64_t)x * h + k];
            raw[n].m = (uint64_t)e[i].w * scale;
            n++;
        }
    }
    qsort(raw, (size_t)n, sizeof(nm_pair), cmp_nm);
    int64_t u = 0;
    for (int64_t i = 0; i < n; i++) {
        if (u > 0 && raw[u - 1].node == raw[i].node) raw[u - 1].m += raw[i].m;
        else raw[u++] = raw[i];
    }
    *out = raw;
    return u;
}

/* QT value.  num = Σ_{v != root} ω(v)·|m_μ(v) − m_ν(v)|, ω(v) = 2^{D* − depth(v)} (integer
 * form of the edge weight 2^{ℓ(v)}, ℓ(v) = ℓ_root − depth(v)); QT = (num · 2^{ℓ_root − D*}) / (W·U). */
int or_qt(const or_tree* T, const int32_t* mu_ids, const uint32_t* mu_w, int32_t s_mu,
          const int32_t* nu_ids, const uint32_t* nu_w, int32_t s_nu, uint64_t* num_out, double* val_out) {
    or_entry *a = NULL, *b = NULL;
    uint64_t W = 0, U = 0;
    int rc = load_support(T, mu_ids, mu_w, s_mu, &a, &W);
    if (rc) return rc;
    rc = load_support(T, nu_ids, nu_w, s_nu, &b, &U);
    if (rc) { free(a); return rc; }
    nm_pair *ma = NULL, *mb = NULL;
    int64_t na = node_masses(T, a, s_mu, U, &ma);
    int64_t nb = node_masses(T, b, s_nu, W, &mb);
    uint64_t num = 0;
    int64_t i = 0, j = 0;
    while (i < na || j < nb) {
        int32_t v; uint64_t x = 0, y = 0;
        if (j >= nb || (i < na && ma[i].node < mb[j].node)) { v = ma[i].node; x = ma[i].m; i++; }
        else if (i >= na || mb[j].node < ma[i].node) { v = mb[j].node; y = mb[j].m; j++; }
        else { v = ma[i].node; x = ma[i].m; y = mb[j].m; i++; j++; }
        uint64_t diff = (x > y) ? (x - y) : (y - x);
        uint64_t omega = (uint64_t)1 << (T->d_star - T->node_depth[v]);
        num += omega * diff;
    }
    free(a); free(b); free(ma); free(mb);
    if (num >= ((uint64_t)1 << 53)) return OR_EOVERFLOW;
    *num_out = num;
    double scaled = ldexp((double)num, T->l_root - T->d_star);
    *val_out = scaled / (double)(W * U);
    return OR_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* O8: greedy bottom-up flow with the canonical tie-break (reading R10):     */
/* at every node, deepest first and in node-ID order, the residual μ- and ν-lists (ids under v */
/* with residual > 0, ascending vocab id) are matched by the two-pointer northwest corner; the */
/* leftover passes up.  Every node, leaves included, matches maximally (reading R8).           */
/* ------------------------------------------------------------------------------------------ */
typedef struct { int32_t depth; int32_t node; } dn_pair;
static int cmp_dn(const void* a, const void* b) {
    const dn_pair* x = (const dn_pair*)a; const dn_pair* y = (const dn_pair*)b;
    if (x->depth != y->depth) return (x->depth > y->depth) ? -1 : 1;   /* depth descending */
    return (x->node < y->node) ? -1 : (x->node > y->node);             /* node id ascending */
}

/* emits triples (src = μ vocab id, dst = ν vocab id, mass η, node where matched) in emission
 * order.  cap bounds the output; returns OR_ECAP if exceeded.                                */
int or_flow(const or_tree* T, const int32_t* mu_ids, const uint32_t* mu_w, int32_t s_mu,
            const int32_t* nu_ids, const uint32_t* nu_w, int32_t s_nu,
            int32_t* src, int32_t* dst, uint64_t* mass, int32_t* node_out, int32_t cap, int32_t* n_out,
            uint64_t* W_out, uint64_t* U_out) {
    or_entry *a = NULL, *b = NULL;
    uint64_t W = 0, U = 0;
    int rc = load_support(T, mu_ids, mu_w, s_mu, &a, &W);
    if (rc) return rc;
    rc = load_support(T, nu_ids, nu_w, s_nu, &b, &U);
    if (rc) { free(a); return rc; }
    int32_t h = T->d_star + 1;
    /* O6: residuals start at the cross-scaled masses */
    uint64_t* ra = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)s_mu);
    uint64_t* rb = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)s_nu);
    for (int32_t i = 0; i < s_mu; i++) ra[i] = (uint64_t)a[i].w * U;
    for (int32_t j = 0; j < s_nu; j++) rb[j] = (uint64_t)b[j].w * W;
    /* nodes with C_μ(v) ∪ C_ν(v) non-empty */
    int64_t cn = 0;
    dn_pair* nodes = (dn_pair*)malloc(sizeof(dn_pair) * ((size_t)(s_mu + s_nu) * (size_t)h));
    for (int32_t i = 0; i < s_mu; i++)
        for (int32_t k = 0; k <= T->leaf_depth[a[i].id]; k++) {
            nodes[cn].depth = k; nodes[cn].node = T->path[(int64_t)a[i].id * h + k]; cn++;
        }
    for (int32_t j = 0; j < s_nu; j++)
        for (int32_t k = 0; k <= T->leaf_depth[b[j].id]; k++) {
            nodes[cn].depth = k; nodes[cn].node = T->path[(int64_t)b[j].id * h + k]; cn++;
        }
    qsort(nodes, (size_t)cn, sizeof(dn_pair), cmp_dn);
    int32_t* la = (int32_t*)malloc(sizeof(int32_t) * (size_t)s_mu);
    int32_t* lb = (int32_t*)malloc(sizeof(int32_t) * (size_t)s_nu);
    int32_t n = 0;
    for (int64_t t = 0; t < cn; t++) {
        if (t > 0 && nodes[t].node == nodes[t - 1].node) continue;   /* unique */
        int32_t k = nodes[t].depth, v = nodes[t].node;
        /* Step 1: collect the unmatched demands under v, ascending vocab id */
        int32_t pa = 0, pb = 0;
        for (int32_t i = 0; i < s_mu; i++)
            if (T->leaf_depth[a[i].id] >= k && T->path[(int64_t)a[i].id * h + k] == v && ra[i] > 0) la[pa++] = i;
        for (int32_t j = 0; j < s_nu; j++)
            if (T->leaf_depth[b[j].id] >= k && T->path[(int64_t)b[j].id * h + k] == v && rb[j] > 0) lb[pb++] = j;
        /* Step 2: while a pair with positive demands exists, match η = min (two-pointer) */
        int32_t x = 0, y = 0;
        while (x < pa && y < pb) {
            uint64_t eta = ra[la[x]] < rb[lb[y]] ? ra[la[x]] : rb[lb[y]];
            if (n >= cap) { rc = OR_ECAP; goto done; }
            src[n] = a[la[x]].id; dst[n] = b[lb[y]].id; mass[n] = eta;
            if (node_out) node_out[n] = v;
            n++;
            ra[la[x]] -= eta; rb[lb[y]] -= eta;
            if (ra[la[x]] == 0) x++;
            if (rb[lb[y]] == 0) y++;
        }
        /* Step 3: the leftover (one side only) passes to the parent implicitly via ra/rb */
    }
    /* after the root every residual is zero */
    for (int32_t i = 0; i < s_mu; i++) if (ra[i] != 0) rc = OR_EINVAL;
    for (int32_t j = 0; j < s_nu; j++) if (rb[j] != 0) rc = OR_EINVAL;
done:
    *n_out = n;
    if (W_out) *W_out = W;
    if (U_out) *U_out = U;
    free(a); free(b); free(ra); free(rb); free(nodes); free(la); free(lb);
    return rc;
}

/* O9: dist(x, y) = sqrt(Σ_i ((double)x_i − (double)y_i)^2), summed in i order; 0 if x = y. */
double or_dist(const float* X, int32_t d, int32_t x, int32_t y) {
    if (x == y) return 0.0;
    double s = 0.0;
    for (int32_t i = 0; i < d; i++) {
        double t = (double)X[(int64_t)x * d + i] - (double)X[(int64_t)y * d + i];
        s = s + t * t;
    }
    return sqrt(s);
}

/* FT = (Σ over triples, in emission order, of (double)η · dist) / (double)(W·U) */
int or_ft(const or_tree* T, const float* X, const int32_t* mu_ids, const uint32_t* mu_w, int32_t s_mu,
          const int32_t* nu_ids, const uint32_t* nu_w, int32_t s_nu, double* val_out) {
    int32_t cap = s_mu + s_nu;
    int32_t* src = (int32_t*)malloc(sizeof(int32_t) * (size_t)cap);
    int32_t* dst = (int32_t*)malloc(sizeof(int32_t) * (size_t)cap);
    uint64_t* mass = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)cap);
    int32_t n = 0; uint64_t W = 0, U = 0;
    int rc = or_flow(T, mu_ids, mu_w, s_mu, nu_ids, nu_w, s_nu, src, dst, mass, NULL, cap, &n, &W, &U);
    if (rc == OR_OK) {
        double acc = 0.0;
        for (int32_t t = 0; t < n; t++) acc = acc + (double)mass[t] * or_dist(X, T->d, src[t], dst[t]);
        *val_out = acc / (double)(W * U);
    }
    free(src); free(dst); free(mass);
    return rc;
}

/* ------------------------------------------------------------------------------------------ */
/* O10: k-NN for one query and the 2-stage prefetch-and-prune pipeline          */
/* Quadtree -> keep m -> Flowtree -> keep k.  Ranks by (value, id).     */
/* ------------------------------------------------------------------------------------------ */
typedef struct { double v; int64_t id; } vi_pair;
static int cmp_vi(const void* a, const void* b) {
    const vi_pair* x = (const vi_pair*)a; const vi_pair* y = (const vi_pair*)b;
    if (x->v < y->v) return -1;
    if (x->v > y->v) return 1;
    return (x->id < y->id) ? -1 : (x->id > y->id);
}

int or_knn(const or_tree* T, const float* X, const int64_t* doc_off, int64_t n, const int32_t* ids,
           const uint32_t* w, const int32_t* q_ids, const uint32_t* q_w, int32_t s_q, int32_t k,
           int64_t prefilter_m, int64_t* out_ids, double* out_val) {
    if (k < 1) return OR_EINVAL;
    if (prefilter_m > 0 && prefilter_m < k) return OR_EINVAL;
    vi_pair* all = (vi_pair*)malloc(sizeof(vi_pair) * (size_t)n);
    int64_t cand_n = n;
    int rc = OR_OK;
    int exhaustive = (prefilter_m <= 0 || prefilter_m >= n);
    if (exhaustive) {
        for (int64_t i = 0; i < n; i++) {
            double v;
            rc = or_ft(T, X, ids + doc_off[i], w + doc_off[i], (int32_t)(doc_off[i + 1] - doc_off[i]),
                       q_ids, q_w, s_q, &v);
            if (rc) goto out;
            all[i].v = v; all[i].id = i;
        }
    } else {
        for (int64_t i = 0; i < n; i++) {
            double v; uint64_t num;
            rc = or_qt(T, ids + doc_off[i], w + doc_off[i], (int32_t)(doc_off[i + 1] - doc_off[i]),
                       q_ids, q_w, s_q, &num, &v);
            if (rc) goto out;
            all[i].v = v; all[i].id = i;
        }
        qsort(all, (size_t)n, sizeof(vi_pair), cmp_vi);
        cand_n = prefilter_m;
        for (int64_t c = 0; c < cand_n; c++) {
            int64_t i = all[c].id;
            double v;
            rc = or_ft(T, X, ids + doc_off[i], w + doc_off[i], (int32_t)(doc_off[i + 1] - doc_off[i]),
                       q_ids, q_w, s_q, &v);
            if (rc) goto out;
            all[c].v = v;
        }
    }
    qsort(all, (size_t)cand_n, sizeof(vi_pair), cmp_vi);
    for (int32_t t = 0; t < k; t++) {
        if (t < cand_n) { out_ids[t] = all[t].id; out_val[t] = all[t].v; }
        else { out_ids[t] = -1; out_val[t] = INFINITY; }
    }
out:
    free(all);
    return rc;
}
