/*
 * pd_oracle.c -- CPU double-precision brute-force oracle for 3D power / Voronoi cells.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  It shares no code, header, table or helper with the
 * CUDA path (paper_2605_06408_b200/csrc) and neither side includes or links the other.
 *
 * What it computes is the plain definition (§3 Eq. 1) restricted to the box
 * (App. "Initialization"), written out as in SURVEY.md §8(c):
 *
 *   H_ij = { x : |x-p_i|^2 - w_i <= |x-p_j|^2 - w_j }
 *        = { y = x-p_i : y.D <= (|D|^2 + w_i - w_j)/2 },  D = p_j - p_i       (Eq. 1, pairwise)
 *   K_i  = B  ∩  ⋂_{j != i} H_ij                                              (cell in the box)
 *   vol_i = |K_i|,  a_ij = area(K_i ∩ ∂H_ij),  N_i = { j : a_ij > 0 } ascending  ("share a
 *   polygonal face")
 *
 * Algorithm (the naive "clip by every bisecting plane" of PAPER.md:196, §4.1):
 *   1. P = B as 6 face loops (ordered vertex lists, outward normals), in site-local coordinates.
 *   2. For every j != i: if the plane's distance from p_i, d_ij = (|D|^2 + w_i - w_j)/(2|D|)
 *      (§4.2), is >= R_max (1 + 1e-12), with R_max the largest |v| over the
 *      current vertices, no vertex can lie outside (v.D <= |v||D| <= R_max |D|): skip.  This is an
 *      exact implication, not a culling heuristic.  Otherwise classify every vertex
 *      (outside <=> v.D - (|D|^2+w_i-w_j)/2 > tau, tau = 1e-13 |D| R_max: on-plane vertices are
 *      kept), clip every face loop (Sutherland-Hodgman), and chain the cut
 *      segments into the new face loop tagged j.
 *      Order: in exact arithmetic K_i does not depend on the order of the intersections; for speed
 *      the `order_k` nearest sites are clipped first (ascending |D|), then every site in index
 *      order.  order_k = 0 gives plain index order (tests check both agree).
 *   3. Face area by Newell's formula, vol = 1/3 sum_f A_f . c_f, S_i = sum of all face areas
 *      (walls included); neighbours = bisector faces with area > 1e-13 S_i, ascending (a smaller
 *      "area" is the FP64 rounding residue of a zero-area edge/vertex contact of a degenerate,
 *      e.g. cospherical, configuration: DESIGN.md reading R2 / SURVEY.md §8(c) Q2).
 *   Coincident sites (bit-identical FP32 positions): the heavier owns, ties go
 *   to the lower id; the other cell is EMPTY|DUPLICATE (Eq. 1: its cell is the empty set).
 *
 * Inputs are the same FP32 arrays the GPU receives, promoted exactly to double.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_EMPTY 1
#define ORC_BOUNDARY 2
#define ORC_OVERFLOW 4
#define ORC_DUPLICATE 8
#define ORC_DEGRADED 16

typedef struct { double x, y, z; } v3;

static inline v3 v3make(double x, double y, double z) { v3 r = {x, y, z}; return r; }
static inline v3 v3sub(v3 a, v3 b) { return v3make(a.x - b.x, a.y - b.y, a.z - b.z); }
static inline v3 v3add(v3 a, v3 b) { return v3make(a.x + b.x, a.y + b.y, a.z + b.z); }
static inline v3 v3scale(v3 a, double s) { return v3make(a.x * s, a.y * s, a.z * s); }
static inline double v3dot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static inline v3 v3cross(v3 a, v3 b) {
    return v3make(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static inline int v3eq(v3 a, v3 b) { return a.x == b.x && a.y == b.y && a.z == b.z; }

typedef struct {
    int tag;        /* >= 0: neighbour site id; -1-k: box wall k (0:-x 1:+x 2:-y 3:+y 4:-z 5:+z) */
    v3 n;           /* plane  n.y <= d  (site-local coordinates) */
    double d;
    int off, nv;    /* loop = verts[off .. off+nv), counter-clockwise seen from outside */
} face_t;

typedef struct {
    face_t* f; int nf, capf;
    v3* v; int nv, capv;
} poly_t;

static void poly_reserve(poly_t* p, int nf, int nv) {
    if (nf > p->capf) { p->capf = nf * 2 + 16; p->f = (face_t*)realloc(p->f, sizeof(face_t) * p->capf); }
    if (nv > p->capv) { p->capv = nv * 2 + 64; p->v = (v3*)realloc(p->v, sizeof(v3) * p->capv); }
}
static void poly_free(poly_t* p) { free(p->f); free(p->v); memset(p, 0, sizeof(*p)); }

/* Box B as six CCW (seen from outside) face loops, local to site s. */
static void poly_init_box(poly_t* p, const double box[6], v3 s) {
    double lo[3] = {box[0] - s.x, box[1] - s.y, box[2] - s.z};
    double hi[3] = {box[3] - s.x, box[4] - s.y, box[5] - s.z};
    v3 c[8];
    for (int k = 0; k < 8; ++k)
        c[k] = v3make((k & 1) ? hi[0] : lo[0], (k & 2) ? hi[1] : lo[1], (k & 4) ? hi[2] : lo[2]);
    static const int loops[6][4] = {{0, 4, 6, 2}, {1, 3, 7, 5}, {0, 1, 5, 4},
                                    {2, 6, 7, 3}, {0, 2, 3, 1}, {4, 5, 7, 6}};
    poly_reserve(p, 6, 24);
    p->nf = 6; p->nv = 24;
    for (int f = 0; f < 6; ++f) {
        int ax = f / 2, pos = f & 1;
        v3 n = v3make(0, 0, 0);
        if (ax == 0) n.x = pos ? 1 : -1;
        if (ax == 1) n.y = pos ? 1 : -1;
        if (ax == 2) n.z = pos ? 1 : -1;
        p->f[f].tag = -1 - f;
        p->f[f].n = n;
        p->f[f].d = pos ? hi[ax] : -lo[ax];
        p->f[f].off = 4 * f;
        p->f[f].nv = 4;
        for (int k = 0; k < 4; ++k) p->v[4 * f + k] = c[loops[f][k]];
    }
}

static double poly_rmax2(const poly_t* p) {
    double r = 0;
    for (int k = 0; k < p->nv; ++k) { double q = v3dot(p->v[k], p->v[k]); if (q > r) r = q; }
    return r;
}

/* Intersection of segment (in, out) with the plane; canonical argument order so that the two
 * faces sharing an edge produce bit-identical points. */
static inline v3 isect(v3 pin, double sin_, v3 pout, double sout) {
    double t = sin_ / (sin_ - sout);
    return v3add(pin, v3scale(v3sub(pout, pin), t));
}

typedef struct { v3 a, b; } seg_t;

/* Clip p by {y : n.y <= d} (tag); result into q.  Returns 0 unchanged (q untouched), 1 clipped,
 * 2 emptied; sets *degraded on a chaining failure. */
static int poly_clip(const poly_t* p, poly_t* q, v3 n, double d, int tag, double tau,
                     seg_t** segs, int* segcap, v3** scratch, int* scap, int* degraded) {
    int any_out = 0;
    for (int k = 0; k < p->nv && !any_out; ++k)
        if (v3dot(n, p->v[k]) - d > tau) any_out = 1;
    if (!any_out) return 0;
    poly_reserve(q, p->nf + 1, 2 * p->nv + 64);
    q->nf = 0; q->nv = 0;
    int nseg = 0;
    for (int f = 0; f < p->nf; ++f) {
        const face_t* F = &p->f[f];
        const v3* V = p->v + F->off;
        int nout = 0;
        for (int k = 0; k < F->nv; ++k) if (v3dot(n, V[k]) - d > tau) ++nout;
        if (q->nf + 1 > q->capf || q->nv + 2 * F->nv + 8 > q->capv)
            poly_reserve(q, q->nf + 2, q->nv + 2 * F->nv + 8);
        face_t* G = &q->f[q->nf];
        *G = *F;
        G->off = q->nv;
        if (nout == 0) {
            memcpy(q->v + q->nv, V, sizeof(v3) * F->nv);
            q->nv += F->nv;
            q->nf++;
            continue;
        }
        int m = 0;
        v3 A = v3make(0, 0, 0);
        int haveA = 0;
        for (int k = 0; k < F->nv; ++k) {
            v3 P = V[k], Q = V[(k + 1) % F->nv];
            double sP = v3dot(n, P) - d, sQ = v3dot(n, Q) - d;
            int cP = sP > tau ? 1 : (sP < -tau ? -1 : 0);   /* 1 out, 0 on, -1 in */
            int cQ = sQ > tau ? 1 : (sQ < -tau ? -1 : 0);
            if (cP != 1) q->v[q->nv + m++] = P;
            if (cP != 1 && cQ == 1) {            /* leaving the kept region: point A */
                if (cP == -1) { A = isect(P, sP, Q, sQ); q->v[q->nv + m++] = A; }
                else A = P;
                haveA = 1;
            } else if (cP == 1 && cQ != 1) {     /* re-entering: point B, edge A->B lies on the plane */
                v3 B;
                if (cQ == -1) { B = isect(Q, sQ, P, sP); q->v[q->nv + m++] = B; }
                else B = Q;
                if (nseg + 1 > *segcap) { *segcap = 2 * nseg + 16; *segs = (seg_t*)realloc(*segs, sizeof(seg_t) * *segcap); }
                (*segs)[nseg].a = B;           /* the new face runs B -> A (opposite orientation) */
                (*segs)[nseg].b = A;
                (*segs)[nseg].a = B;
                if (!haveA) {                  /* run started before vertex 0: A fixed up below */
                    (*segs)[nseg].b = v3make(NAN, NAN, NAN);
                }
                nseg++;
                haveA = 0;
            }
        }
        if (haveA) {
            /* the out-run wraps around the end of the loop: its B was recorded first with a NaN A */
            int fixed = 0;
            for (int s = nseg - 1; s >= 0; --s)
                if (isnan((*segs)[s].b.x)) { (*segs)[s].b = A; fixed = 1; break; }
            if (!fixed) *degraded = 1;
        }
        if (m >= 3) { G->nv = m; q->nv += m; q->nf++; }
    }
    /* drop zero-length segments (plane touching at a single vertex) */
    int ns = 0;
    for (int s = 0; s < nseg; ++s) {
        if (isnan((*segs)[s].b.x)) { *degraded = 1; continue; }
        if (!v3eq((*segs)[s].a, (*segs)[s].b)) (*segs)[ns++] = (*segs)[s];
    }
    if (q->nf == 0) return 2;
    if (ns >= 3) {
        if (ns + 1 > *scap) { *scap = 2 * ns + 16; *scratch = (v3*)realloc(*scratch, sizeof(v3) * *scap); }
        v3* L = *scratch;
        int* used = (int*)calloc(ns, sizeof(int));
        int m = 0;
        L[m++] = (*segs)[0].a;
        v3 cur = (*segs)[0].b;
        used[0] = 1;
        int closed = 0;
        for (int it = 0; it < ns; ++it) {
            if (v3eq(cur, L[0])) { closed = 1; break; }
            int found = -1;
            for (int s = 0; s < ns; ++s)
                if (!used[s] && v3eq((*segs)[s].a, cur)) { found = s; break; }
            if (found < 0) break;
            used[found] = 1;
            L[m++] = cur;
            cur = (*segs)[found].b;
        }
        for (int s = 0; s < ns; ++s) if (!used[s]) *degraded = 1;
        if (!closed) *degraded = 1;
        if (m >= 3) {
            poly_reserve(q, q->nf + 1, q->nv + m);
            face_t* H = &q->f[q->nf++];
            H->tag = tag; H->n = n; H->d = d; H->off = q->nv; H->nv = m;
            memcpy(q->v + q->nv, L, sizeof(v3) * m);
            q->nv += m;
        }
        free(used);
    }
    return 1;
}

/* ---------------------------------------------------------------------------------------------- */

typedef struct {
    const float* pts; const float* w; int64_t n; double box[6];
    int order_k;
} orc_input;

typedef struct {
    int nf;
    int* tags; double* areas; /* per face (incl. walls) */
    double vol, surf;
    int flags;
    int32_t* nbr; double* nbr_area; int nnbr;
    int n_dropped;  /* bisector faces with area <= 1e-13 S (zero-area contacts, not neighbours: R2) */
    int n_small;    /* neighbour faces with area < 1e-9 S (near-degenerate: BASELINE north_star) */
    /* geometry (optional) */
    poly_t geo;
} orc_cell;

static inline v3 site(const orc_input* in, int64_t j) {
    return v3make((double)in->pts[3 * j], (double)in->pts[3 * j + 1], (double)in->pts[3 * j + 2]);
}
static inline double wt(const orc_input* in, int64_t j) { return in->w ? (double)in->w[j] : 0.0; }

typedef struct { double key; int64_t j; } kn_t;

static void heap_sift_down(kn_t* h, int n, int i) {
    for (;;) {
        int l = 2 * i + 1, r = l + 1, m = i;
        if (l < n && h[l].key > h[m].key) m = l;
        if (r < n && h[r].key > h[m].key) m = r;
        if (m == i) return;
        kn_t t = h[i]; h[i] = h[m]; h[m] = t; i = m;
    }
}
static int kn_cmp(const void* a, const void* b) {
    double x = ((const kn_t*)a)->key, y = ((const kn_t*)b)->key;
    if (x < y) return -1;
    if (x > y) return 1;
    int64_t p = ((const kn_t*)a)->j, q = ((const kn_t*)b)->j;
    return (p > q) - (p < q);
}
static int tagarea_cmp(const void* a, const void* b) {
    const double* x = (const double*)a; const double* y = (const double*)b;
    return (x[0] > y[0]) - (x[0] < y[0]);
}

typedef struct {
    poly_t P[2];
    seg_t* segs; int segcap;
    v3* scratch; int scap;
    kn_t* heap; int heapcap;
} orc_ws;

static void ws_free(orc_ws* ws) {
    poly_free(&ws->P[0]); poly_free(&ws->P[1]);
    free(ws->segs); free(ws->scratch); free(ws->heap);
    memset(ws, 0, sizeof(*ws));
}

/* Build cell i.  Returns the index (0/1) of the final polyhedron in ws->P, -1 if empty. */
static int build_cell(const orc_input* in, int64_t i, orc_ws* ws, int* flags) {
    v3 pi = site(in, i);
    double wi = wt(in, i);
    int cur = 0;
    int degraded = 0;
    *flags = 0;
    poly_init_box(&ws->P[cur], in->box, pi);
    double rmax2 = poly_rmax2(&ws->P[cur]);
    /* --- ordering pass: the order_k nearest sites first (speed only) --- */
    int K = in->order_k;
    if (K > in->n - 1) K = (int)(in->n - 1);
    int nh = 0;
    if (K > 0) {
        if (ws->heapcap < K) { ws->heapcap = K; ws->heap = (kn_t*)realloc(ws->heap, sizeof(kn_t) * K); }
        for (int64_t j = 0; j < in->n; ++j) {
            if (j == i) continue;
            v3 D = v3sub(site(in, j), pi);
            double q = v3dot(D, D);
            if (nh < K) {
                ws->heap[nh].key = q; ws->heap[nh].j = j; nh++;
                if (nh == K) for (int s = K / 2 - 1; s >= 0; --s) heap_sift_down(ws->heap, K, s);
            } else if (q < ws->heap[0].key) {
                ws->heap[0].key = q; ws->heap[0].j = j; heap_sift_down(ws->heap, K, 0);
            }
        }
        qsort(ws->heap, nh, sizeof(kn_t), kn_cmp);
    }
    for (int pass = 0; pass < 2; ++pass) {
        int64_t cnt = pass == 0 ? nh : in->n;
        for (int64_t t = 0; t < cnt; ++t) {
            int64_t j = pass == 0 ? ws->heap[t].j : t;
            if (j == i) continue;
            v3 pj = site(in, j);
            double wj = wt(in, j);
            v3 D = v3sub(pj, pi);
            double D2 = v3dot(D, D);
            if (D2 == 0.0) {
                /* coincident sites (Q5): heavier owns, ties to the lower id */
                if (wj > wi || (wj == wi && j < i)) { *flags |= ORC_EMPTY | ORC_DUPLICATE; return -1; }
                continue;
            }
            double dd = 0.5 * (D2 + wi - wj);          /* plane: y.D <= dd */
            double nD = sqrt(D2);
            double dij = dd / nD;
            double rmax = sqrt(rmax2);
            if (dij >= rmax * (1.0 + 1e-12)) continue;   /* exact implication: nothing outside */
            double tau = 1e-13 * nD * rmax;
            int r = poly_clip(&ws->P[cur], &ws->P[cur ^ 1], D, dd, (int)j, tau,
                              &ws->segs, &ws->segcap, &ws->scratch, &ws->scap, &degraded);
            if (r == 0) continue;
            cur ^= 1;
            if (r == 2) { *flags |= ORC_EMPTY; if (degraded) *flags |= ORC_DEGRADED; return -1; }
            rmax2 = poly_rmax2(&ws->P[cur]);
        }
    }
    if (degraded) *flags |= ORC_DEGRADED;
    return cur;
}

static void finalize_cell(const poly_t* p, orc_cell* out, int flags) {
    out->flags = flags;
    out->vol = 0; out->surf = 0; out->nnbr = 0; out->nf = 0; out->n_dropped = 0; out->n_small = 0;
    if (!p) { out->flags |= ORC_EMPTY; return; }
    out->nf = p->nf;
    out->tags = (int*)malloc(sizeof(int) * (p->nf + 1));
    out->areas = (double*)malloc(sizeof(double) * (p->nf + 1));
    double* ta = (double*)malloc(sizeof(double) * 2 * (p->nf + 1));
    int nt = 0;
    double vol = 0, surf = 0;
    for (int f = 0; f < p->nf; ++f) {
        const face_t* F = &p->f[f];
        const v3* V = p->v + F->off;
        v3 A = v3make(0, 0, 0), c = v3make(0, 0, 0);
        for (int k = 0; k < F->nv; ++k) {
            A = v3add(A, v3cross(V[k], V[(k + 1) % F->nv]));   /* Newell */
            c = v3add(c, V[k]);
        }
        A = v3scale(A, 0.5);
        c = v3scale(c, 1.0 / F->nv);
        double area = sqrt(v3dot(A, A));
        vol += v3dot(A, c) / 3.0;
        surf += area;
        out->tags[f] = F->tag;
        out->areas[f] = area;
    }
    double amin = 1e-13 * surf;   /* zero-area contacts: reading R2 */
    for (int f = 0; f < p->nf; ++f) {
        double area = out->areas[f];
        if (out->tags[f] < 0) { if (area > amin) out->flags |= ORC_BOUNDARY; }
        else if (area > amin) {
            ta[2 * nt] = (double)out->tags[f]; ta[2 * nt + 1] = area; nt++;
            if (area < 1e-9 * surf) out->n_small++;
        } else out->n_dropped++;
    }
    qsort(ta, nt, 2 * sizeof(double), tagarea_cmp);
    out->nbr = (int32_t*)malloc(sizeof(int32_t) * (nt + 1));
    out->nbr_area = (double*)malloc(sizeof(double) * (nt + 1));
    int m = 0;
    for (int k = 0; k < nt; ++k) {
        int32_t t = (int32_t)ta[2 * k];
        if (m > 0 && out->nbr[m - 1] == t) { out->nbr_area[m - 1] += ta[2 * k + 1]; out->flags |= ORC_DEGRADED; continue; }
        out->nbr[m] = t; out->nbr_area[m] = ta[2 * k + 1]; m++;
    }
    out->nnbr = m;
    out->vol = vol;
    out->surf = surf;
    if (!(vol > 0)) out->flags |= ORC_EMPTY;
    free(ta);
}

/* ------------------------------- public (ctypes) entry points -------------------------------- */

typedef struct {
    int64_t ncells;
    orc_cell* cells;
} orc_result;

typedef struct {
    const orc_input* in;
    const int64_t* ids;
    int64_t ncells;
    orc_cell* out;
    int64_t next;
    pthread_mutex_t mu;
} orc_job;

static void* worker(void* arg) {
    orc_job* job = (orc_job*)arg;
    orc_ws ws;
    memset(&ws, 0, sizeof(ws));
    for (;;) {
        pthread_mutex_lock(&job->mu);
        int64_t t = job->next++;
        pthread_mutex_unlock(&job->mu);
        if (t >= job->ncells) break;
        int flags = 0;
        int r = build_cell(job->in, job->ids[t], &ws, &flags);
        finalize_cell(r >= 0 ? &ws.P[r] : NULL, &job->out[t], flags);
    }
    ws_free(&ws);
    return NULL;
}

int orc_version(void) { return 1; }

/* Build the cells ids[0..ncells) of the diagram of (pts, w) in box.  w may be NULL (Voronoi).
 * box = {lo.x, lo.y, lo.z, hi.x, hi.y, hi.z}.  Returns NULL on allocation failure. */
orc_result* orc_run(const float* pts, const float* w, int64_t n, const double* box,
                    const int64_t* ids, int64_t ncells, int nthreads, int order_k) {
    orc_input in;
    in.pts = pts; in.w = w; in.n = n; in.order_k = order_k;
    memcpy(in.box, box, sizeof(in.box));
    orc_result* res = (orc_result*)calloc(1, sizeof(orc_result));
    res->ncells = ncells;
    res->cells = (orc_cell*)calloc(ncells > 0 ? ncells : 1, sizeof(orc_cell));
    orc_job job;
    job.in = &in; job.ids = ids; job.ncells = ncells; job.out = res->cells; job.next = 0;
    pthread_mutex_init(&job.mu, NULL);
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, worker, &job);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    pthread_mutex_destroy(&job.mu);
    return res;
}

int64_t orc_nnz(const orc_result* r) {
    int64_t s = 0;
    for (int64_t t = 0; t < r->ncells; ++t) s += r->cells[t].nnbr;
    return s;
}

/* offsets[ncells+1], nbr[nnz], area[nnz], vol[ncells], surf[ncells], flags[ncells] */
void orc_copy(const orc_result* r, int64_t* offsets, int32_t* nbr, double* area, double* vol,
              double* surf, uint8_t* flags) {
    int64_t o = 0;
    for (int64_t t = 0; t < r->ncells; ++t) {
        const orc_cell* c = &r->cells[t];
        offsets[t] = o;
        for (int k = 0; k < c->nnbr; ++k) { nbr[o + k] = c->nbr[k]; area[o + k] = c->nbr_area[k]; }
        o += c->nnbr;
        vol[t] = c->vol; surf[t] = c->surf; flags[t] = (uint8_t)c->flags;
    }
    offsets[r->ncells] = o;
}

/* per cell: dropped[t] = bisector faces with area <= 1e-13 S, small[t] = neighbour faces < 1e-9 S */
void orc_counts(const orc_result* r, int32_t* dropped, int32_t* small) {
    for (int64_t t = 0; t < r->ncells; ++t) { dropped[t] = r->cells[t].n_dropped; small[t] = r->cells[t].n_small; }
}

void orc_free(orc_result* r) {
    if (!r) return;
    for (int64_t t = 0; t < r->ncells; ++t) {
        free(r->cells[t].tags); free(r->cells[t].areas);
        free(r->cells[t].nbr); free(r->cells[t].nbr_area);
    }
    free(r->cells);
    free(r);
}

/* Geometry of one cell, for the pins that need vertices (empty power sphere, ownership).
 * Writes up to max_faces faces: tag[f], nverts[f], plane[4f..4f+3] = (n, d) in LOCAL coords, and
 * the loops' vertices in WORLD coordinates into xyz (3 doubles each, up to max_verts).
 * Returns the number of faces (0 if empty), or -1 if capacities are too small. */
int orc_cell_geometry(const float* pts, const float* w, int64_t n, const double* box, int64_t i,
                      int order_k, int max_faces, int max_verts, int* tags, int* nverts,
                      double* planes, double* xyz, int* flags_out) {
    orc_input in;
    in.pts = pts; in.w = w; in.n = n; in.order_k = order_k;
    memcpy(in.box, box, sizeof(in.box));
    orc_ws ws;
    memset(&ws, 0, sizeof(ws));
    int flags = 0;
    int r = build_cell(&in, i, &ws, &flags);
    *flags_out = flags;
    if (r < 0) { ws_free(&ws); return 0; }
    const poly_t* p = &ws.P[r];
    if (p->nf > max_faces || p->nv > max_verts) { ws_free(&ws); return -1; }
    v3 pi = site(&in, i);
    int o = 0;
    for (int f = 0; f < p->nf; ++f) {
        tags[f] = p->f[f].tag;
        nverts[f] = p->f[f].nv;
        planes[4 * f] = p->f[f].n.x; planes[4 * f + 1] = p->f[f].n.y;
        planes[4 * f + 2] = p->f[f].n.z; planes[4 * f + 3] = p->f[f].d;
        for (int k = 0; k < p->f[f].nv; ++k) {
            v3 v = v3add(p->v[p->f[f].off + k], pi);
            xyz[3 * o] = v.x; xyz[3 * o + 1] = v.y; xyz[3 * o + 2] = v.z; o++;
        }
    }
    int nf = p->nf;
    ws_free(&ws);
    return nf;
}

/* ==============================================================================================
 * CPU reference of the same definition (a reported baseline, NOT the oracle the
 * parity tests use).  The oracle's clipper above, fed by a best-first walk of a k-d tree whose every
 * subtree carries its bounding box and the largest weight in it (the CPU analogue of the paper's
 * weight-augmented BVH), and stopped by the radius of security (prior work,
 * PAPER.md:126, :221) in its weighted form:
 *   a site j at distance D >= d from p_i with w_j <= w_max has its plane at distance
 *   d_ij = (D^2 + w_i - w_j)/(2D) >= f(D) = (D^2 + c)/(2D), c = w_i - w_max
 *   and min_{D >= d} f(D) = f(d) if c <= 0 or d^2 >= c, else sqrt(c)  (f decreases up to sqrt(c)).
 * Subtrees are visited in ascending order of that lower bound; once it reaches R_max (1 + 1e-12), no
 * remaining site can cut the cell -- the same implication as build_cell's exact skip.  Exact arithmetic
 * gives the oracle's polytope (clip order is irrelevant); rounding differs, so the tests compare the two
 * with the comparator's tolerances.  Multithreaded over cells; the tree is built once per point set.
 * ============================================================================================== */

typedef struct {
    orc_input in;
    int32_t* idx;      /* permutation of 0..n-1, kd-ordered; subtree [b,e) is keyed by its mid (b+e)/2 */
    int32_t* axis;     /* per key: split axis */
    double* bb;        /* per key: bounding box of the subtree's sites (lo.xyz, hi.xyz) */
    double* wmax;      /* per key: largest weight in the subtree */
} orc_kd;

static double coord(const orc_input* in, int32_t j, int ax) { return (double)in->pts[3 * (int64_t)j + ax]; }

static void kd_build_rec(orc_kd* t, int64_t b, int64_t e) {
    if (e <= b) return;
    int64_t mid = (b + e) / 2;
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    double wm = -1e300;
    for (int64_t k = b; k < e; ++k) {
        for (int a = 0; a < 3; ++a) {
            double v = coord(&t->in, t->idx[k], a);
            if (v < lo[a]) lo[a] = v;
            if (v > hi[a]) hi[a] = v;
        }
        double wk = wt(&t->in, t->idx[k]);
        if (wk > wm) wm = wk;
    }
    int ax = 0;
    for (int a = 1; a < 3; ++a) if (hi[a] - lo[a] > hi[ax] - lo[ax]) ax = a;
    /* quickselect the median on axis ax (ties broken by index: deterministic) */
    int64_t l = b, r = e - 1;
    while (l < r) {
        int32_t piv = t->idx[(l + r) / 2];
        double pv = coord(&t->in, piv, ax);
        int64_t i = l, j = r;
        while (i <= j) {
            while (coord(&t->in, t->idx[i], ax) < pv || (coord(&t->in, t->idx[i], ax) == pv && t->idx[i] < piv)) ++i;
            while (coord(&t->in, t->idx[j], ax) > pv || (coord(&t->in, t->idx[j], ax) == pv && t->idx[j] > piv)) --j;
            if (i <= j) { int32_t s = t->idx[i]; t->idx[i] = t->idx[j]; t->idx[j] = s; ++i; --j; }
        }
        if (mid <= j) r = j; else if (mid >= i) l = i; else break;
    }
    t->axis[mid] = ax;
    for (int a = 0; a < 3; ++a) { t->bb[6 * mid + a] = lo[a]; t->bb[6 * mid + 3 + a] = hi[a]; }
    t->wmax[mid] = wm;
    kd_build_rec(t, b, mid);
    kd_build_rec(t, mid + 1, e);
}

/* Lower bound of the plane distance d_ij over the subtree keyed `key` (see the header above). */
static double kd_lower_bound(const orc_kd* t, int64_t key, v3 pi, double wi) {
    const double* bb = t->bb + 6 * key;
    double q[3] = {pi.x, pi.y, pi.z}, d2 = 0;
    for (int a = 0; a < 3; ++a) {
        double g = q[a] < bb[a] ? bb[a] - q[a] : (q[a] > bb[3 + a] ? q[a] - bb[3 + a] : 0.0);
        d2 += g * g;
    }
    double c = wi - t->wmax[key];
    if (c > 0 && d2 < c) return sqrt(c);
    if (d2 == 0) return -HUGE_VAL;
    return (d2 + c) / (2.0 * sqrt(d2));
}

typedef struct { double lb; int64_t b, e; } kd_ent;
typedef struct { kd_ent* h; int64_t n, cap; } kd_heap;   /* min-heap on lb */

static void kdh_push(kd_heap* H, kd_ent x) {
    if (H->n == H->cap) { H->cap = H->cap ? 2 * H->cap : 256; H->h = (kd_ent*)realloc(H->h, sizeof(kd_ent) * H->cap); }
    int64_t i = H->n++;
    while (i > 0) { int64_t p = (i - 1) / 2; if (H->h[p].lb <= x.lb) break; H->h[i] = H->h[p]; i = p; }
    H->h[i] = x;
}
static kd_ent kdh_pop(kd_heap* H) {
    kd_ent top = H->h[0], x = H->h[--H->n];
    int64_t i = 0;
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, m = i;
        double best = x.lb;
        if (l < H->n && H->h[l].lb < best) { m = l; best = H->h[l].lb; }
        if (r < H->n && H->h[r].lb < best) { m = r; }
        if (m == i) break;
        H->h[i] = H->h[m]; i = m;
    }
    if (H->n > 0) H->h[i] = x;
    return top;
}

typedef struct {
    const orc_kd* tree;
    const int64_t* ids;
    int64_t ncells;
    orc_cell* out;
    int64_t next;
    pthread_mutex_t mu;
} kd_job;

static int build_cell_kd(const orc_kd* tree, int64_t i, orc_ws* ws, kd_heap* H, int* flags) {
    const orc_input* in = &tree->in;
    v3 pi = site(in, i);
    double wi = wt(in, i);
    int cur = 0, degraded = 0;
    *flags = 0;
    poly_init_box(&ws->P[cur], in->box, pi);
    double rmax = sqrt(poly_rmax2(&ws->P[cur]));
    H->n = 0;
    if (in->n > 0) { kd_ent root = {kd_lower_bound(tree, in->n / 2, pi, wi), 0, in->n}; kdh_push(H, root); }
    while (H->n > 0) {
        kd_ent x = kdh_pop(H);
        if (x.lb >= rmax * (1.0 + 1e-12)) break;   /* radius of security: no remaining site can cut */
        int64_t mid = (x.b + x.e) / 2;
        if (mid > x.b) { kd_ent l = {kd_lower_bound(tree, (x.b + mid) / 2, pi, wi), x.b, mid}; kdh_push(H, l); }
        if (x.e > mid + 1) { kd_ent r = {kd_lower_bound(tree, (mid + 1 + x.e) / 2, pi, wi), mid + 1, x.e}; kdh_push(H, r); }
        int64_t j = tree->idx[mid];
        if (j == i) continue;
        v3 D = v3sub(site(in, j), pi);
        double D2 = v3dot(D, D);
        double wj = wt(in, j);
        if (D2 == 0.0) {   /* coincident sites (Q5) */
            if (wj > wi || (wj == wi && j < i)) { *flags |= ORC_EMPTY | ORC_DUPLICATE; return -1; }
            continue;
        }
        double nD = sqrt(D2);
        double dd = 0.5 * (D2 + wi - wj);
        if (dd / nD >= rmax * (1.0 + 1e-12)) continue;   /* the oracle's exact skip */
        double tau = 1e-13 * nD * rmax;
        int r = poly_clip(&ws->P[cur], &ws->P[cur ^ 1], D, dd, (int)j, tau,
                          &ws->segs, &ws->segcap, &ws->scratch, &ws->scap, &degraded);
        if (r == 0) continue;
        cur ^= 1;
        if (r == 2) { *flags |= ORC_EMPTY; if (degraded) *flags |= ORC_DEGRADED; return -1; }
        rmax = sqrt(poly_rmax2(&ws->P[cur]));
    }
    if (degraded) *flags |= ORC_DEGRADED;
    return cur;
}

static void* kd_worker(void* arg) {
    kd_job* job = (kd_job*)arg;
    orc_ws ws;
    memset(&ws, 0, sizeof(ws));
    kd_heap H = {NULL, 0, 0};
    for (;;) {
        pthread_mutex_lock(&job->mu);
        int64_t t0 = job->next;
        job->next += 64;
        pthread_mutex_unlock(&job->mu);
        if (t0 >= job->ncells) break;
        int64_t t1 = t0 + 64 < job->ncells ? t0 + 64 : job->ncells;
        for (int64_t t = t0; t < t1; ++t) {
            int flags = 0;
            int r = build_cell_kd(job->tree, job->ids[t], &ws, &H, &flags);
            finalize_cell(r >= 0 ? &ws.P[r] : NULL, &job->out[t], flags);
        }
    }
    free(H.h);
    ws_free(&ws);
    return NULL;
}

/* Build the tree once per point set (the arrays are borrowed and must outlive the handle). */
orc_kd* orc_kd_build(const float* pts, const float* w, int64_t n, const double* box) {
    orc_kd* t = (orc_kd*)calloc(1, sizeof(orc_kd));
    t->in.pts = pts; t->in.w = w; t->in.n = n; t->in.order_k = 0;
    memcpy(t->in.box, box, sizeof(t->in.box));
    int64_t m = n > 0 ? n : 1;
    t->idx = (int32_t*)malloc(sizeof(int32_t) * m);
    t->axis = (int32_t*)calloc(m, sizeof(int32_t));
    t->bb = (double*)malloc(sizeof(double) * 6 * m);
    t->wmax = (double*)malloc(sizeof(double) * m);
    for (int64_t j = 0; j < n; ++j) t->idx[j] = (int32_t)j;
    kd_build_rec(t, 0, n);
    return t;
}

void orc_kd_free(orc_kd* t) {
    if (!t) return;
    free(t->idx); free(t->axis); free(t->bb); free(t->wmax); free(t);
}

/* Cells ids[0..ncells) from a built tree; same outputs as orc_run (orc_nnz / orc_copy / orc_counts / orc_free). */
orc_result* orc_kd_run(const orc_kd* tree, const int64_t* ids, int64_t ncells, int nthreads) {
    orc_result* res = (orc_result*)calloc(1, sizeof(orc_result));
    res->ncells = ncells;
    res->cells = (orc_cell*)calloc(ncells > 0 ? ncells : 1, sizeof(orc_cell));
    kd_job job;
    job.tree = tree; job.ids = ids; job.ncells = ncells; job.out = res->cells; job.next = 0;
    pthread_mutex_init(&job.mu, NULL);
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, kd_worker, &job);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    pthread_mutex_destroy(&job.mu);
    return res;
}

orc_result* orc_run_kdtree(const float* pts, const float* w, int64_t n, const double* box, const int64_t* ids,
                           int64_t ncells, int nthreads) {
    orc_kd* t = orc_kd_build(pts, w, n, box);
    orc_result* r = orc_kd_run(t, ids, ncells, nthreads);
    orc_kd_free(t);
    return r;
}
