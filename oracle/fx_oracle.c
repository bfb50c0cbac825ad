/* TEST INFRASTRUCTURE -- NOT PART OF THE PRODUCT.
 *
 * Plain-C restatement of the reference featurex hot path, used only as the
 * parity checker (see fx_oracle.h).  Each function names the reference lines it
 * follows (paths relative to /root/reference/proj).  Floating-point expressions
 * keep the reference's operation order and are compiled with
 * -ffp-contract=off, so most columns agree bit for bit with the reference; the
 * pinning tests (tests/test_oracle_pin.py) measure that agreement against the
 * compiled reference itself.
 */
#include "fx_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* fxo_last_error(void) { return g_err; }

typedef struct {
    uint32_t x, y;
    uint16_t v;
} px_t;

typedef struct {
    uint32_t xmin, ymin, xmax, ymax; /* inclusive, roi.hpp:20-26 */
} bbox_t;

typedef struct {
    const px_t* p;
    size_t n;
    bbox_t bb;
} cloud_t;

/* ---------------------------------------------------------------- columns -- */

/* feature_columns (engine.cpp:107-136): intensity 39 (intensity_features.cpp:217-234),
 * shape 38, moments 104 (moments.cpp:96-115), glcm 29 per angle + _ave
 * (texture.cpp:534-542), glrlm 16 per angle + _ave, glszm 16, ngtdm 5. */
int fxo_n_cols(unsigned groups, const fxo_params* p) {
    const int a = p->n_angles;
    int n = 0;
    if (groups & FXO_INTENSITY) n += 39;
    if (groups & FXO_SHAPE) n += 38;
    if (groups & FXO_MOMENTS) n += 104;
    if (groups & FXO_GLCM) n += 29 * (a + 1);
    if (groups & FXO_GLRLM) n += 16 * (a + 1);
    if (groups & FXO_GLSZM) n += 16;
    if (groups & FXO_NGTDM) n += 5;
    return n;
}

/* ------------------------------------------------------------ label scan -- */

/* RoiRegistry::accumulate (roi.cpp:76-110): first pixel seeds the bbox, then
 * min/max; labels() ascending (roi.cpp:112-117). */
int fxo_roi_table(const uint16_t* labels, int w, int h, uint32_t* out_labels,
                  uint64_t* out_count, uint32_t* out_bbox, size_t cap, size_t* n) {
    uint64_t* cnt = calloc(65536, sizeof(uint64_t));
    bbox_t* bb = calloc(65536, sizeof(bbox_t));
    if (!cnt || !bb) {
        free(cnt);
        free(bb);
        return fail(8, "oom");
    }
    for (int y = 0; y < h; ++y) {
        for (int x = 0; x < w; ++x) {
            const uint16_t l = labels[(size_t)y * w + x];
            if (!l) continue;
            if (cnt[l] == 0) {
                bb[l].xmin = bb[l].xmax = (uint32_t)x;
                bb[l].ymin = bb[l].ymax = (uint32_t)y;
            } else {
                if ((uint32_t)x < bb[l].xmin) bb[l].xmin = (uint32_t)x;
                if ((uint32_t)x > bb[l].xmax) bb[l].xmax = (uint32_t)x;
                if ((uint32_t)y < bb[l].ymin) bb[l].ymin = (uint32_t)y;
                if ((uint32_t)y > bb[l].ymax) bb[l].ymax = (uint32_t)y;
            }
            cnt[l]++;
        }
    }
    size_t k = 0;
    for (int l = 1; l < 65536; ++l) {
        if (!cnt[l]) continue;
        if (k < cap) {
            out_labels[k] = (uint32_t)l;
            out_count[k] = cnt[l];
            out_bbox[4 * k + 0] = bb[l].xmin;
            out_bbox[4 * k + 1] = bb[l].ymin;
            out_bbox[4 * k + 2] = bb[l].xmax;
            out_bbox[4 * k + 3] = bb[l].ymax;
        }
        ++k;
    }
    *n = k;
    free(cnt);
    free(bb);
    return k > cap ? fail(10, "capacity") : 0;
}

/* --------------------------------------------------------------- contour -- */

/* Moore ring, contour.cpp:13-14 */
static const int kRing[8][2] = {{-1, 0}, {-1, -1}, {0, -1}, {1, -1},
                                {1, 0},  {1, 1},   {0, 1},  {-1, 1}};

typedef struct {
    int w, h, x0, y0;
    uint8_t* cells;
} grid_t;

static int g_at(const grid_t* g, int x, int y) {
    if (x < 0 || x >= g->w || y < 0 || y >= g->h) return 0;
    return g->cells[(size_t)y * g->w + x] != 0;
}

/* keep_largest_component (contour.cpp:30-66): 8-connected flood fill, largest
 * kept, ties -> first found in row-major scan. */
static int keep_largest_component(grid_t* g) {
    const size_t cells = (size_t)g->w * g->h;
    int* comp = calloc(cells, sizeof(int));
    int* stack = malloc(cells * 8 * 2 * sizeof(int) + 16);
    if (!comp || !stack) {
        free(comp);
        free(stack);
        return 8;
    }
    int next = 0, best = 0;
    size_t best_size = 0;
    for (int y = 0; y < g->h; ++y) {
        for (int x = 0; x < g->w; ++x) {
            if (!g_at(g, x, y) || comp[(size_t)y * g->w + x] != 0) continue;
            ++next;
            size_t size = 0, sp = 0;
            stack[sp++] = x;
            stack[sp++] = y;
            comp[(size_t)y * g->w + x] = next;
            while (sp) {
                const int cy = stack[--sp];
                const int cx = stack[--sp];
                ++size;
                for (int k = 0; k < 8; ++k) {
                    const int nx = cx + kRing[k][0], ny = cy + kRing[k][1];
                    if (!g_at(g, nx, ny)) continue;
                    int* c = &comp[(size_t)ny * g->w + nx];
                    if (*c == 0) {
                        *c = next;
                        stack[sp++] = nx;
                        stack[sp++] = ny;
                    }
                }
            }
            if (size > best_size) {
                best_size = size;
                best = next;
            }
        }
    }
    if (next > 1)
        for (size_t i = 0; i < cells; ++i)
            if (g->cells[i] && comp[i] != best) g->cells[i] = 0;
    free(comp);
    free(stack);
    return 0;
}

/* trace_contour (contour.cpp:70-144).  Returns malloc'd interleaved x,y. */
static int trace_contour(const cloud_t* c, int32_t** out_xy, size_t* n_points) {
    *out_xy = NULL;
    *n_points = 0;
    if (c->n == 0) return 0;
    grid_t g;
    g.x0 = (int)c->bb.xmin;
    g.y0 = (int)c->bb.ymin;
    g.w = (int)(c->bb.xmax - c->bb.xmin) + 1;
    g.h = (int)(c->bb.ymax - c->bb.ymin) + 1;
    const size_t cells = (size_t)g.w * g.h;
    g.cells = calloc(cells, 1);
    if (!g.cells) return 8;
    for (size_t i = 0; i < c->n; ++i)
        g.cells[(size_t)((int)c->p[i].y - g.y0) * g.w + ((int)c->p[i].x - g.x0)] = 1;
    if (keep_largest_component(&g)) {
        free(g.cells);
        return 8;
    }
    int sx = -1, sy = -1;
    for (int y = 0; y < g.h && sx < 0; ++y)
        for (int x = 0; x < g.w; ++x)
            if (g_at(&g, x, y)) {
                sx = x;
                sy = y;
                break;
            }
    /* state (pos, backtrack) -> first walk index (the unordered_map of :98-106) */
    int64_t* seen = malloc(cells * 8 * sizeof(int64_t));
    const size_t max_steps = 8 * cells + 16;
    int32_t* walk = malloc((max_steps + 1) * 2 * sizeof(int32_t));
    if (!seen || !walk) {
        free(seen);
        free(walk);
        free(g.cells);
        return 8;
    }
    for (size_t i = 0; i < cells * 8; ++i) seen[i] = -1;
    int cx = sx, cy = sy, back = 0;
    size_t nw = 0, cycle_start = 0;
    for (size_t step = 0; step < max_steps; ++step) {
        const size_t state = ((size_t)cy * g.w + cx) * 8 + (size_t)back;
        if (seen[state] >= 0) {
            cycle_start = (size_t)seen[state];
            break;
        }
        seen[state] = (int64_t)nw;
        walk[2 * nw] = cx + g.x0;
        walk[2 * nw + 1] = cy + g.y0;
        ++nw;
        int found = -1;
        for (int k = 1; k <= 8; ++k) {
            const int idx = (back + k) % 8;
            if (g_at(&g, cx + kRing[idx][0], cy + kRing[idx][1])) {
                found = idx;
                break;
            }
        }
        if (found < 0) break;
        const int prev = (found + 7) % 8;
        const int bx = cx + kRing[prev][0], by = cy + kRing[prev][1];
        cx += kRing[found][0];
        cy += kRing[found][1];
        for (int k = 0; k < 8; ++k)
            if (cx + kRing[k][0] == bx && cy + kRing[k][1] == by) {
                back = k;
                break;
            }
    }
    const size_t np = nw - cycle_start;
    int32_t* pts = malloc((np ? np : 1) * 2 * sizeof(int32_t));
    memcpy(pts, walk + 2 * cycle_start, np * 2 * sizeof(int32_t));
    *out_xy = pts;
    *n_points = np;
    free(seen);
    free(walk);
    free(g.cells);
    return 0;
}

/* ------------------------------------------------------------- intensity -- */

static int cmp_double(const void* a, const void* b) {
    const double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}

/* percentile / median_of (intensity_features.cpp:14-27) */
static double percentile(const double* s, size_t n, double p) {
    if (n == 1) return s[0];
    const double rank = p / 100.0 * (double)(n - 1);
    const size_t lo = (size_t)rank;
    if (lo + 1 >= n) return s[n - 1];
    const double frac = rank - (double)lo;
    return s[lo] + frac * (s[lo + 1] - s[lo]);
}

static double median_of(const double* s, size_t n) {
    return n % 2 ? s[n / 2] : 0.5 * (s[n / 2 - 1] + s[n / 2]);
}

/* intensity_features (intensity_features.cpp:42-215), values in the order of
 * intensity_feature_values (:236-276). */
static int intensity_group(const cloud_t* c, int bins, double* out) {
    memset(out, 0, 39 * sizeof(double));
    const size_t n = c->n;
    if (n == 0) return 0;
    double* v = malloc(n * sizeof(double));
    double* s = malloc(n * sizeof(double));
    double* devs = malloc(n * sizeof(double));
    if (!v || !s || !devs) {
        free(v);
        free(s);
        free(devs);
        return 8;
    }
    for (size_t i = 0; i < n; ++i) v[i] = (double)c->p[i].v;
    memcpy(s, v, n * sizeof(double));
    qsort(s, n, sizeof(double), cmp_double);

    const double dn = (double)n;
    double sum = 0;
    for (size_t i = 0; i < n; ++i) sum += v[i];
    const double mean = sum / dn;
    const double mn = s[0], mx = s[n - 1], range = mx - mn;
    const double median = median_of(s, n);

    double m2 = 0, m3 = 0, m4 = 0, m5 = 0, m6 = 0;
    for (size_t i = 0; i < n; ++i) {
        const double d = v[i] - mean;
        const double d2 = d * d;
        m2 += d2;
        m3 += d2 * d;
        m4 += d2 * d2;
        m5 += d2 * d2 * d;
        m6 += d2 * d2 * d2;
    }
    m2 /= dn;
    m3 /= dn;
    m4 /= dn;
    m5 /= dn;
    m6 /= dn;
    const double variance_biased = m2;
    const double variance = n > 1 ? m2 * dn / (dn - 1.0) : 0.0;
    const double std_biased = sqrt(variance_biased);
    const double std_dev = sqrt(variance);
    double skew = 0, kurt = 0, exkurt = 0, hskew = 0, hflat = 0;
    if (m2 > 0) {
        skew = m3 / pow(m2, 1.5);
        kurt = m4 / (m2 * m2);
        exkurt = kurt - 3.0;
        hskew = m5 / pow(m2, 2.5);
        hflat = m6 / (m2 * m2 * m2);
    }
    double mad = 0;
    for (size_t i = 0; i < n; ++i) mad += fabs(v[i] - mean);
    mad = mad / dn;

    for (size_t i = 0; i < n; ++i) devs[i] = fabs(s[i] - median);
    qsort(devs, n, sizeof(double), cmp_double);
    const double median_ad = median_of(devs, n);

    const double p1 = percentile(s, n, 1), p10 = percentile(s, n, 10);
    const double p25 = percentile(s, n, 25), p75 = percentile(s, n, 75);
    const double p90 = percentile(s, n, 90), p99 = percentile(s, n, 99);
    const double iqr = p75 - p25;
    const double qcod = (p75 + p25) != 0 ? iqr / (p75 + p25) : 0.0;

    double rmad = 0;
    {
        double rsum = 0;
        size_t rn = 0;
        for (size_t i = 0; i < n; ++i)
            if (s[i] >= p10 && s[i] <= p90) {
                rsum += s[i];
                ++rn;
            }
        if (rn > 0) {
            const double rmean = rsum / (double)rn;
            double acc = 0;
            for (size_t i = 0; i < n; ++i)
                if (s[i] >= p10 && s[i] <= p90) acc += fabs(s[i] - rmean);
            rmad = acc / (double)rn;
        }
    }
    double mode = s[0];
    {
        size_t best_run = 0, i = 0;
        while (i < n) {
            size_t j = i;
            while (j < n && s[j] == s[i]) ++j;
            if (j - i > best_run) {
                best_run = j - i;
                mode = s[i];
            }
            i = j;
        }
    }
    double energy = 0;
    for (size_t i = 0; i < n; ++i) energy += v[i] * v[i];
    const double rms = sqrt(energy / dn);
    const double cov = mean != 0 ? std_dev / mean : 0.0;

    double entropy = 0, uniformity = 0;
    {
        const int nb = bins > 2 ? bins : 2;
        size_t* hist = calloc((size_t)nb, sizeof(size_t));
        if (range == 0) {
            hist[0] = n;
        } else {
            for (size_t i = 0; i < n; ++i) {
                int b = (int)((double)nb * (v[i] - mn) / range);
                if (b >= nb) b = nb - 1;
                ++hist[b];
            }
        }
        for (int b = 0; b < nb; ++b) {
            if (hist[b] == 0) continue;
            const double p = (double)hist[b] / dn;
            entropy -= p * log2(p);
            uniformity += p * p;
        }
        free(hist);
    }

    double edge_mean = 0, edge_min = 0, edge_max = 0, edge_std = 0, edge_int = 0;
    {
        int32_t* pts = NULL;
        size_t np = 0;
        if (trace_contour(c, &pts, &np)) {
            free(v);
            free(s);
            free(devs);
            return 8;
        }
        const int w = (int)(c->bb.xmax - c->bb.xmin) + 1;
        const int h = (int)(c->bb.ymax - c->bb.ymin) + 1;
        uint8_t* on = calloc((size_t)w * h, 1);
        for (size_t i = 0; i < np; ++i)
            on[(size_t)(pts[2 * i + 1] - (int)c->bb.ymin) * w + (pts[2 * i] - (int)c->bb.xmin)] = 1;
        double es = 0, emin = 0, emax = 0;
        size_t en_ = 0;
        for (size_t i = 0; i < n; ++i) {
            const px_t* q = &c->p[i];
            if (!on[(size_t)(q->y - c->bb.ymin) * w + (q->x - c->bb.xmin)]) continue;
            const double x = (double)q->v;
            if (en_ == 0) emin = emax = x;
            es += x;
            if (x < emin) emin = x;
            if (x > emax) emax = x;
            ++en_;
        }
        if (en_) {
            const double en = (double)en_;
            edge_mean = es / en;
            edge_min = emin;
            edge_max = emax;
            edge_int = es;
            double ev = 0;
            for (size_t i = 0; i < n; ++i) {
                const px_t* q = &c->p[i];
                if (!on[(size_t)(q->y - c->bb.ymin) * w + (q->x - c->bb.xmin)]) continue;
                const double x = (double)q->v;
                ev += (x - edge_mean) * (x - edge_mean);
            }
            edge_std = sqrt(ev / en);
        }
        free(on);
        free(pts);
    }

    /* weighted_centroid (:31-40) guarded by isum > 0 (:205-213) */
    double wcx = 0, wcy = 0;
    {
        double isum = 0, sx = 0, sy = 0;
        for (size_t i = 0; i < n; ++i) isum += c->p[i].v;
        if (isum > 0) {
            for (size_t i = 0; i < n; ++i) {
                sx += (double)c->p[i].x * c->p[i].v;
                sy += (double)c->p[i].y * c->p[i].v;
            }
            wcx = sx / isum;
            wcy = sy / isum;
        }
    }

    const double vals[39] = {mean,      median,   mode,     mn,        mx,       range,
                             variance,  variance_biased,    std_dev,   std_biased,
                             mad,       median_ad, rmad,    iqr,       p1,       p10,
                             p25,       p75,      p90,      p99,       skew,     kurt,
                             exkurt,    hskew,    hflat,    energy,    rms,      entropy,
                             uniformity, qcod,    cov,      sum,       edge_mean, edge_min,
                             edge_max,  edge_std, edge_int, wcx,       wcy};
    memcpy(out, vals, sizeof vals);
    free(v);
    free(s);
    free(devs);
    return 0;
}

/* --------------------------------------------------------------- moments -- */

static const double kBinom[4][4] = {{1, 0, 0, 0}, {1, 1, 0, 0}, {1, 2, 1, 0}, {1, 3, 3, 1}};

typedef struct {
    double raw[4][4], central[4][4], eta[4][4], hu[7];
} moments_t;

/* hu_from_eta (moments.cpp:14-28) */
static void hu_from_eta(const double eta[4][4], double hu[7]) {
    const double n20 = eta[2][0], n02 = eta[0][2], n11 = eta[1][1];
    const double n30 = eta[3][0], n03 = eta[0][3], n21 = eta[2][1], n12 = eta[1][2];
    const double a = n30 + n12;
    const double b = n21 + n03;
    hu[0] = n20 + n02;
    hu[1] = (n20 - n02) * (n20 - n02) + 4.0 * n11 * n11;
    hu[2] = (n30 - 3.0 * n12) * (n30 - 3.0 * n12) + (3.0 * n21 - n03) * (3.0 * n21 - n03);
    hu[3] = a * a + b * b;
    hu[4] = (n30 - 3.0 * n12) * a * (a * a - 3.0 * b * b) +
            (3.0 * n21 - n03) * b * (3.0 * a * a - b * b);
    hu[5] = (n20 - n02) * (a * a - b * b) + 4.0 * n11 * a * b;
    hu[6] = (3.0 * n21 - n03) * a * (a * a - 3.0 * b * b) -
            (n30 - 3.0 * n12) * b * (3.0 * a * a - b * b);
}

/* compute_moments (moments.cpp:32-92); returns 6 (ZeroMassError) for a
 * zero-mass weighted cloud. */
static int compute_moments(const cloud_t* c, int weighted, moments_t* m) {
    memset(m, 0, sizeof *m);
    if (c->n == 0) return 0;
    const double x0 = c->bb.xmin, y0 = c->bb.ymin;
    double local[4][4];
    memset(local, 0, sizeof local);
    for (size_t k = 0; k < c->n; ++k) {
        const px_t* p = &c->p[k];
        const double w = weighted ? (double)p->v : 1.0;
        double xp = 1.0, lxp = 1.0;
        for (int i = 0; i <= 3; ++i) {
            double yq = 1.0, lyq = 1.0;
            for (int j = 0; j <= 3; ++j) {
                m->raw[i][j] += w * xp * yq;
                local[i][j] += w * lxp * lyq;
                yq *= (double)p->y;
                lyq *= (double)p->y - y0;
            }
            xp *= (double)p->x;
            lxp *= (double)p->x - x0;
        }
    }
    const double m00 = m->raw[0][0];
    if (weighted && m00 <= 0.0) return 6;
    if (m00 == 0.0) return 0;
    const double lcx = local[1][0] / m00;
    const double lcy = local[0][1] / m00;
    for (int p = 0; p <= 3; ++p)
        for (int q = 0; q <= 3; ++q) {
            double acc = 0.0;
            for (int i = 0; i <= p; ++i)
                for (int j = 0; j <= q; ++j)
                    acc += kBinom[p][i] * kBinom[q][j] * pow(-lcx, p - i) * pow(-lcy, q - j) *
                           local[i][j];
            m->central[p][q] = acc;
        }
    m->central[1][0] = 0.0;
    m->central[0][1] = 0.0;
    for (int p = 0; p <= 3; ++p)
        for (int q = 0; q <= 3; ++q) {
            if (p + q < 2) continue;
            m->eta[p][q] = m->central[p][q] / pow(m00, 1.0 + (p + q) / 2.0);
        }
    hu_from_eta(m->eta, m->hu);
    return 0;
}

/* append_moment_values (moments.cpp:117-129) */
static double* append_moments(const moments_t* m, double* out) {
    for (int p = 0; p <= 3; ++p)
        for (int q = 0; q <= 3; ++q) *out++ = m->raw[p][q];
    for (int p = 0; p <= 3; ++p)
        for (int q = 0; q <= 3; ++q) *out++ = m->central[p][q];
    for (int p = 0; p <= 3; ++p)
        for (int q = 0; q <= 3; ++q)
            if (p + q >= 2) *out++ = m->eta[p][q];
    for (int k = 0; k < 7; ++k) *out++ = m->hu[k];
    return out;
}

/* --------------------------------------------------------------- texture -- */

typedef struct {
    int w, h, x0, y0, ng;
    int16_t* grid; /* level or -1 */
} droi_t;

/* discretize (texture.cpp:29-56) */
static int discretize(const cloud_t* c, int ng, droi_t* r) {
    if (ng < 2) return fail(1, "grey level count must be >= 2");
    r->ng = ng;
    r->x0 = (int)c->bb.xmin;
    r->y0 = (int)c->bb.ymin;
    r->w = (int)(c->bb.xmax - c->bb.xmin) + 1;
    r->h = (int)(c->bb.ymax - c->bb.ymin) + 1;
    const size_t cells = (size_t)r->w * r->h;
    r->grid = malloc(cells * sizeof(int16_t));
    if (!r->grid) return 8;
    for (size_t i = 0; i < cells; ++i) r->grid[i] = -1;
    if (c->n == 0) return 0;
    uint16_t lo = c->p[0].v, hi = lo;
    for (size_t i = 0; i < c->n; ++i) {
        if (c->p[i].v < lo) lo = c->p[i].v;
        if (c->p[i].v > hi) hi = c->p[i].v;
    }
    const double span = (double)hi - lo + 1.0;
    for (size_t i = 0; i < c->n; ++i) {
        int level = 0;
        if (hi > lo) {
            level = (int)((double)ng * (c->p[i].v - lo) / span);
            if (level > ng - 1) level = ng - 1;
        }
        r->grid[(size_t)((int)c->p[i].y - r->y0) * r->w + ((int)c->p[i].x - r->x0)] =
            (int16_t)level;
    }
    return 0;
}

static int d_inside(const droi_t* r, int x, int y) {
    return x >= 0 && x < r->w && y >= 0 && y < r->h && r->grid[(size_t)y * r->w + x] >= 0;
}

/* angle_offset (texture.cpp:15-23) */
static int angle_offset(int angle, int d, int* dx, int* dy) {
    switch (angle) {
        case 0: *dx = d; *dy = 0; return 0;
        case 45: *dx = d; *dy = -d; return 0;
        case 90: *dx = 0; *dy = -d; return 0;
        case 135: *dx = -d; *dy = -d; return 0;
        default: return fail(1, "unsupported angle");
    }
}

/* glcm counting loop (texture.cpp:58-80) */
static int glcm_count(const droi_t* r, int offset, int angle, int symmetric, uint64_t* counts,
                      uint64_t* pairs) {
    int dx = 0, dy = 0;
    if (angle_offset(angle, offset, &dx, &dy)) return 1;
    memset(counts, 0, (size_t)r->ng * r->ng * sizeof(uint64_t));
    *pairs = 0;
    for (int y = 0; y < r->h; ++y)
        for (int x = 0; x < r->w; ++x) {
            if (!d_inside(r, x, y)) continue;
            const int a = r->grid[(size_t)y * r->w + x];
            const int nx = x + dx, ny = y + dy;
            if (!d_inside(r, nx, ny)) continue;
            const int b = r->grid[(size_t)ny * r->w + nx];
            counts[(size_t)a * r->ng + b] += 1;
            if (symmetric) counts[(size_t)b * r->ng + a] += 1;
            *pairs += 1;
        }
    return 0;
}

static double log2_safe(double p) { return p > 0 ? log2(p) : 0.0; }

/* glcm_features (texture.cpp:87-217) on p (ng*ng, normalized as :81-84). */
static void glcm_features(const double* P, int ng, uint64_t pair_count, double out[29]) {
    memset(out, 0, 29 * sizeof(double));
    if (pair_count == 0) return;
    double* px = calloc((size_t)ng, sizeof(double));
    double* py = calloc((size_t)ng, sizeof(double));
    double* pxy = calloc((size_t)(2 * ng - 1), sizeof(double));
    double* pxmy = calloc((size_t)ng, sizeof(double));
    double asm_ = 0, contrast = 0, entropy = 0, idm = 0, id = 0, idn = 0, idmn = 0;
    double iv = 0, dis = 0, acor = 0, jmax = 0;
    for (int a = 0; a < ng; ++a)
        for (int b = 0; b < ng; ++b) {
            const double p = P[(size_t)a * ng + b];
            if (p == 0) continue;
            const double i = a + 1, j = b + 1;
            const double diff = i - j;
            px[a] += p;
            py[b] += p;
            pxy[a + b] += p;
            pxmy[abs(a - b)] += p;
            asm_ += p * p;
            contrast += diff * diff * p;
            entropy -= p * log2(p);
            idm += p / (1.0 + diff * diff);
            id += p / (1.0 + fabs(diff));
            idn += p / (1.0 + fabs(diff) / ng);
            idmn += p / (1.0 + diff * diff / ((double)ng * ng));
            if (a != b) iv += p / (diff * diff);
            dis += fabs(diff) * p;
            acor += i * j * p;
            if (p > jmax) jmax = p;
        }
    double mu_x = 0, mu_y = 0;
    for (int a = 0; a < ng; ++a) {
        mu_x += (a + 1) * px[a];
        mu_y += (a + 1) * py[a];
    }
    double var_x = 0, var_y = 0, hx = 0, hy = 0;
    for (int a = 0; a < ng; ++a) {
        var_x += (a + 1 - mu_x) * (a + 1 - mu_x) * px[a];
        var_y += (a + 1 - mu_y) * (a + 1 - mu_y) * py[a];
        hx -= px[a] * log2_safe(px[a]);
        hy -= py[a] * log2_safe(py[a]);
    }
    double corr = 0;
    if (var_x > 0 && var_y > 0) corr = (acor - mu_x * mu_y) / sqrt(var_x * var_y);
    double clutend = 0, clushade = 0, cluprom = 0, jvar = 0, hxy1 = 0, hxy2 = 0;
    for (int a = 0; a < ng; ++a)
        for (int b = 0; b < ng; ++b) {
            const double p = P[(size_t)a * ng + b];
            const double i = a + 1, j = b + 1;
            const double s = i + j - mu_x - mu_y;
            if (p > 0) {
                clutend += s * s * p;
                clushade += s * s * s * p;
                cluprom += s * s * s * s * p;
                jvar += (i - mu_x) * (i - mu_x) * p;
                hxy1 -= p * log2_safe(px[a] * py[b]);
            }
            if (px[a] > 0 && py[b] > 0) hxy2 -= px[a] * py[b] * log2(px[a] * py[b]);
        }
    double sumave = 0, sument = 0;
    for (int k = 0; k < 2 * ng - 1; ++k) {
        const double p = pxy[k];
        if (p == 0) continue;
        sumave += (k + 2) * p;
        sument -= p * log2(p);
    }
    double sumvar = 0;
    for (int k = 0; k < 2 * ng - 1; ++k)
        if (pxy[k] > 0) sumvar += (k + 2 - sumave) * (k + 2 - sumave) * pxy[k];
    double difave = 0, difentro = 0;
    for (int k = 0; k < ng; ++k) {
        const double p = pxmy[k];
        if (p == 0) continue;
        difave += k * p;
        difentro -= p * log2(p);
    }
    double difvar = 0;
    for (int k = 0; k < ng; ++k)
        if (pxmy[k] > 0) difvar += (k - difave) * (k - difave) * pxmy[k];
    const double hmax = hx > hy ? hx : hy;
    const double infomeas1 = hmax > 0 ? (entropy - hxy1) / hmax : 0.0;
    const double t = 1.0 - exp(-2.0 * (hxy2 - entropy));
    const double infomeas2 = sqrt(t > 0.0 ? t : 0.0);
    const double v[29] = {asm_,    acor,     cluprom,  clushade, clutend, contrast,  corr,
                          difave,  difentro, difvar,   dis,      sqrt(asm_), entropy, id,
                          idm,     id,       idn,      idm,      idmn,    infomeas1, infomeas2,
                          iv,      mu_x,     entropy,  jmax,     jvar,    sumave,    sument,
                          sumvar};
    memcpy(out, v, sizeof v);
    free(px);
    free(py);
    free(pxy);
    free(pxmy);
}

static int cmp_int(const void* a, const void* b) {
    return (*(const int*)a > *(const int*)b) - (*(const int*)a < *(const int*)b);
}

/* glcm group: per sorted angle glcm -> glcm_features, then emit_per_angle
 * (engine.cpp:159-169, 191-196). */
static int glcm_group(const cloud_t* c, const fxo_params* prm, double* out) {
    droi_t r;
    memset(&r, 0, sizeof r);
    int rc = discretize(c, prm->ng, &r);
    if (rc) return rc;
    const int A = prm->n_angles;
    int angles[8];
    memcpy(angles, prm->angles, (size_t)A * sizeof(int));
    qsort(angles, (size_t)A, sizeof(int), cmp_int);
    const size_t ng2 = (size_t)prm->ng * prm->ng;
    uint64_t* counts = malloc(ng2 * sizeof(uint64_t));
    double* P = malloc(ng2 * sizeof(double));
    double f[8][29];
    for (int a = 0; a < A && !rc; ++a) {
        uint64_t pairs = 0;
        rc = glcm_count(&r, prm->offset, angles[a], prm->symmetric, counts, &pairs);
        if (rc) break;
        const double total = prm->symmetric ? 2.0 * (double)pairs : (double)pairs;
        for (size_t i = 0; i < ng2; ++i) P[i] = pairs ? (double)counts[i] / total : 0.0;
        glcm_features(P, prm->ng, pairs, f[a]);
    }
    if (!rc)
        for (int s = 0; s < 29; ++s) {
            double acc = 0;
            for (int a = 0; a < A; ++a) {
                *out++ = f[a][s];
                acc += f[a][s];
            }
            *out++ = acc / (double)A;
        }
    free(counts);
    free(P);
    free(r.grid);
    return rc;
}

/* ------------------------------------------------- glrlm / glszm / ngtdm -- */

static int d_level(const droi_t* r, int x, int y) { return r->grid[(size_t)y * r->w + x]; }

/* (level, extent) entries -> sorted cells with counts (the reference's std::map
 * iteration order), then the features of glrlm_features (texture.cpp:282-341) /
 * glszm_features (:382-441), which share this form. */
typedef struct {
    int level, extent;
} le_t;

static int cmp_le(const void* a, const void* b) {
    const le_t* p = a;
    const le_t* q = b;
    if (p->level != q->level) return p->level < q->level ? -1 : 1;
    return (p->extent > q->extent) - (p->extent < q->extent);
}

static void grey_count_features(le_t* ent, size_t ne, int ng, uint64_t roi_pixels,
                                double out[16]) {
    memset(out, 0, 16 * sizeof(double));
    if (ne == 0) return;
    qsort(ent, ne, sizeof(le_t), cmp_le);
    /* aggregate in place: cells (level, extent, count) */
    size_t nc = 0;
    uint64_t* cnt = malloc(ne * sizeof(uint64_t));
    int max_ext = 0;
    for (size_t i = 0; i < ne; ++i) {
        if (nc && ent[nc - 1].level == ent[i].level && ent[nc - 1].extent == ent[i].extent) {
            cnt[nc - 1] += 1;
        } else {
            ent[nc] = ent[i];
            cnt[nc++] = 1;
        }
        if (ent[i].extent > max_ext) max_ext = ent[i].extent;
    }
    const double nr = (double)ne, np = (double)roi_pixels;
    double sre = 0, lre = 0, lglre = 0, hglre = 0, srlgle = 0, srhgle = 0, lrlgle = 0, lrhgle = 0;
    double re = 0, glv = 0, rv = 0, mu_g = 0, mu_l = 0;
    double* per_level = calloc((size_t)ng, sizeof(double));
    double* per_len = calloc((size_t)max_ext + 1, sizeof(double));
    for (size_t i = 0; i < nc; ++i) {
        const double r = (double)cnt[i], g = ent[i].level + 1, l = ent[i].extent;
        sre += r / (l * l);
        lre += r * l * l;
        lglre += r / (g * g);
        hglre += r * g * g;
        srlgle += r / (g * g * l * l);
        srhgle += r * g * g / (l * l);
        lrlgle += r * l * l / (g * g);
        lrhgle += r * g * g * l * l;
        per_level[ent[i].level] += r;
        per_len[ent[i].extent] += r;
        const double p = r / nr;
        re -= p * log2(p);
        mu_g += p * g;
        mu_l += p * l;
    }
    for (size_t i = 0; i < nc; ++i) {
        const double p = (double)cnt[i] / nr;
        glv += p * (ent[i].level + 1 - mu_g) * (ent[i].level + 1 - mu_g);
        rv += p * (ent[i].extent - mu_l) * (ent[i].extent - mu_l);
    }
    double glnu = 0, rlnu = 0;
    for (int lv = 0; lv < ng; ++lv)
        if (per_level[lv] != 0) glnu += per_level[lv] * per_level[lv];
    for (int e = 0; e <= max_ext; ++e)
        if (per_len[e] != 0) rlnu += per_len[e] * per_len[e];
    const double v[16] = {sre / nr, lre / nr, glnu / nr, glnu / (nr * nr), rlnu / nr,
                          rlnu / (nr * nr), nr / np, glv, rv, re, lglre / nr, hglre / nr,
                          srlgle / nr, srhgle / nr, lrlgle / nr, lrhgle / nr};
    memcpy(out, v, sizeof v);
    free(cnt);
    free(per_level);
    free(per_len);
}

/* glrlm (texture.cpp:242-280): runs of equal level along the scan direction;
 * a run starts where the predecessor is outside or differs. */
static int glrlm_angle(const droi_t* r, int angle, uint64_t roi_pixels, double out[16]) {
    int dx = 0, dy = 0;
    switch (angle) {
        case 0: dx = 1; dy = 0; break;
        case 45: dx = 1; dy = -1; break;
        case 90: dx = 0; dy = 1; break;
        case 135: dx = 1; dy = 1; break;
        default: return fail(1, "unsupported angle");
    }
    le_t* ent = malloc(((size_t)r->w * r->h + 1) * sizeof(le_t));
    if (!ent) return 8;
    size_t ne = 0;
    for (int y = 0; y < r->h; ++y)
        for (int x = 0; x < r->w; ++x) {
            if (!d_inside(r, x, y)) continue;
            const int g = d_level(r, x, y);
            if (d_inside(r, x - dx, y - dy) && d_level(r, x - dx, y - dy) == g) continue;
            int len = 1, nx = x + dx, ny = y + dy;
            while (d_inside(r, nx, ny) && d_level(r, nx, ny) == g) {
                ++len;
                nx += dx;
                ny += dy;
            }
            ent[ne++] = (le_t){g, len};
        }
    grey_count_features(ent, ne, r->ng, roi_pixels, out);
    free(ent);
    return 0;
}

/* glszm (texture.cpp:343-380): 8-connected zones of equal level, row-major scan */
static int glszm_all(const droi_t* r, uint64_t roi_pixels, double out[16]) {
    const size_t cells = (size_t)r->w * r->h;
    uint8_t* seen = calloc(cells, 1);
    int* st = malloc(cells * 2 * sizeof(int) + 16);
    le_t* ent = malloc((cells + 1) * sizeof(le_t));
    if (!seen || !st || !ent) {
        free(seen);
        free(st);
        free(ent);
        return 8;
    }
    static const int k8[8][2] = {{1, 0}, {-1, 0}, {0, 1}, {0, -1}, {1, 1}, {1, -1}, {-1, 1}, {-1, -1}};
    size_t ne = 0;
    for (int y = 0; y < r->h; ++y)
        for (int x = 0; x < r->w; ++x) {
            if (!d_inside(r, x, y) || seen[(size_t)y * r->w + x]) continue;
            const int g = d_level(r, x, y);
            size_t size = 0, sp = 0;
            st[sp++] = x;
            st[sp++] = y;
            seen[(size_t)y * r->w + x] = 1;
            while (sp) {
                const int cy = st[--sp], cx = st[--sp];
                ++size;
                for (int k = 0; k < 8; ++k) {
                    const int nx = cx + k8[k][0], ny = cy + k8[k][1];
                    if (!d_inside(r, nx, ny) || d_level(r, nx, ny) != g) continue;
                    uint8_t* sn = &seen[(size_t)ny * r->w + nx];
                    if (!*sn) {
                        *sn = 1;
                        st[sp++] = nx;
                        st[sp++] = ny;
                    }
                }
            }
            ent[ne++] = (le_t){g, (int)size};
        }
    grey_count_features(ent, ne, r->ng, roi_pixels, out);
    free(seen);
    free(st);
    free(ent);
    return 0;
}

/* ngtdm + ngtdm_features (texture.cpp:443-528) */
static int ngtdm_all(const droi_t* r, double out[5]) {
    const int ng = r->ng;
    uint64_t* n = calloc((size_t)ng, sizeof(uint64_t));
    double* sv = calloc((size_t)ng, sizeof(double));
    double* p = calloc((size_t)ng, sizeof(double));
    uint64_t valid = 0;
    for (int y = 0; y < r->h; ++y)
        for (int x = 0; x < r->w; ++x) {
            if (!d_inside(r, x, y)) continue;
            double sum = 0;
            int count = 0;
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    if (dx == 0 && dy == 0) continue;
                    if (d_inside(r, x + dx, y + dy)) {
                        sum += d_level(r, x + dx, y + dy) + 1;
                        ++count;
                    }
                }
            if (count == 0) continue;
            const int g = d_level(r, x, y);
            n[g] += 1;
            sv[g] += fabs((g + 1) - sum / count);
            ++valid;
        }
    memset(out, 0, 5 * sizeof(double));
    if (valid) {
        const double nv = (double)valid;
        int present = 0;
        double s_total = 0, ps_total = 0;
        for (int i = 0; i < ng; ++i) {
            p[i] = (double)n[i] / nv;
            if (p[i] > 0) ++present;
            s_total += sv[i];
            ps_total += p[i] * sv[i];
        }
        const double coarseness = ps_total > 0 ? 1.0 / ps_total : 1e6;
        double contrast = 0;
        if (present > 1) {
            double acc = 0;
            for (int i = 0; i < ng; ++i) {
                if (p[i] == 0) continue;
                for (int j = 0; j < ng; ++j) {
                    if (p[j] == 0) continue;
                    acc += p[i] * p[j] * (i - j) * (i - j);
                }
            }
            contrast = acc / ((double)present * (present - 1)) * (s_total / nv);
        }
        double busy = 0, cplx = 0, strn = 0;
        for (int i = 0; i < ng; ++i) {
            if (p[i] == 0) continue;
            const double gi = i + 1;
            for (int j = 0; j < ng; ++j) {
                if (p[j] == 0) continue;
                const double gj = j + 1;
                busy += fabs(gi * p[i] - gj * p[j]);
                cplx += fabs(gi - gj) * (p[i] * sv[i] + p[j] * sv[j]) / (p[i] + p[j]);
                strn += (p[i] + p[j]) * (gi - gj) * (gi - gj);
            }
        }
        out[0] = busy > 0 ? ps_total / busy : 0.0;
        out[1] = coarseness;
        out[2] = cplx / nv;
        out[3] = contrast;
        out[4] = s_total > 0 ? strn / s_total : 0.0;
    }
    free(n);
    free(sv);
    free(p);
    return 0;
}

static int rlzn_groups(const cloud_t* c, unsigned groups, const fxo_params* prm, double** o) {
    droi_t r;
    memset(&r, 0, sizeof r);
    int rc = discretize(c, prm->ng, &r);
    if (rc) return rc;
    if (groups & FXO_GLRLM) {
        const int A = prm->n_angles;
        int angles[8];
        memcpy(angles, prm->angles, (size_t)A * sizeof(int));
        qsort(angles, (size_t)A, sizeof(int), cmp_int);
        double f[8][16];
        for (int a = 0; a < A && !rc; ++a) rc = glrlm_angle(&r, angles[a], c->n, f[a]);
        if (!rc)
            for (int s2 = 0; s2 < 16; ++s2) {
                double acc = 0;
                for (int a = 0; a < A; ++a) {
                    *(*o)++ = f[a][s2];
                    acc += f[a][s2];
                }
                *(*o)++ = acc / (double)A;
            }
    }
    if (!rc && (groups & FXO_GLSZM)) {
        rc = glszm_all(&r, c->n, *o);
        *o += 16;
    }
    if (!rc && (groups & FXO_NGTDM)) {
        rc = ngtdm_all(&r, *o);
        *o += 5;
    }
    free(r.grid);
    return rc;
}

/* ----------------------------------------------------------------- shape -- */

typedef struct {
    int x, y;
} pt_t;

static long long cross3(pt_t o, pt_t a, pt_t b) {
    return (long long)(a.x - o.x) * (b.y - o.y) - (long long)(a.y - o.y) * (b.x - o.x);
}

static int cmp_pt(const void* a, const void* b) {
    const pt_t* p = a;
    const pt_t* q = b;
    if (p->x != q->x) return p->x < q->x ? -1 : 1;
    return (p->y > q->y) - (p->y < q->y);
}

/* convex_hull (hull.cpp:17-55): Andrew's monotone chain over the sorted unique
 * pixel centres, pops on cross <= 0 (collinear points removed); <= 2 points are
 * returned as they are, an all-collinear set as its two end points. */
static int convex_hull(const cloud_t* c, pt_t** out, size_t* nv) {
    pt_t* pts = malloc((c->n ? c->n : 1) * sizeof(pt_t));
    if (!pts) return 8;
    for (size_t i = 0; i < c->n; ++i) pts[i] = (pt_t){(int)c->p[i].x, (int)c->p[i].y};
    qsort(pts, c->n, sizeof(pt_t), cmp_pt);
    size_t n = 0;
    for (size_t i = 0; i < c->n; ++i)
        if (!n || pts[i].x != pts[n - 1].x || pts[i].y != pts[n - 1].y) pts[n++] = pts[i];
    if (n <= 2) {
        *out = pts;
        *nv = n;
        return 0;
    }
    pt_t* h = malloc(2 * n * sizeof(pt_t));
    if (!h) {
        free(pts);
        return 8;
    }
    size_t k = 0;
    for (size_t i = 0; i < n; ++i) {
        while (k >= 2 && cross3(h[k - 2], h[k - 1], pts[i]) <= 0) --k;
        h[k++] = pts[i];
    }
    const size_t lower = k + 1;
    for (size_t i = n - 1; i-- > 0;) {
        while (k >= lower && cross3(h[k - 2], h[k - 1], pts[i]) <= 0) --k;
        h[k++] = pts[i];
    }
    k -= 1;
    if (k < 3) {
        h[0] = pts[0];
        h[1] = pts[n - 1];
        k = 2;
    }
    free(pts);
    *out = h;
    *nv = k;
    return 0;
}

/* point_in_hull (hull.cpp:66-87), eps 1e-9 */
static int point_in_hull(const pt_t* v, size_t nv, double px, double py) {
    const double eps = 1e-9;
    if (nv == 0) return 0;
    if (nv == 1) return fabs(px - v[0].x) < eps && fabs(py - v[0].y) < eps;
    if (nv == 2) {
        const double ax = v[0].x, ay = v[0].y, bx = v[1].x, by = v[1].y;
        const double cr = (bx - ax) * (py - ay) - (by - ay) * (px - ax);
        if (fabs(cr) > eps) return 0;
        const double dot = (px - ax) * (bx - ax) + (py - ay) * (by - ay);
        const double len2 = (bx - ax) * (bx - ax) + (by - ay) * (by - ay);
        return dot >= -eps && dot <= len2 + eps;
    }
    for (size_t i = 0; i < nv; ++i) {
        const pt_t a = v[i], b = v[(i + 1) % nv];
        const double cr = (double)(b.x - a.x) * (py - a.y) - (double)(b.y - a.y) * (px - a.x);
        if (cr < -eps) return 0;
    }
    return 1;
}

/* euler_number (shape_features.cpp:24-99): 8-connected foreground components
 * minus 4-connected background components of the 1-padded bbox grid that do not
 * reach the padding. */
static int euler_number(const cloud_t* c) {
    const int w = (int)(c->bb.xmax - c->bb.xmin) + 3, h = (int)(c->bb.ymax - c->bb.ymin) + 3;
    const int x0 = (int)c->bb.xmin - 1, y0 = (int)c->bb.ymin - 1;
    const size_t cells = (size_t)w * h;
    uint8_t* fg = calloc(cells, 1);
    int* mark = calloc(cells, sizeof(int));
    int* st = malloc(cells * 2 * 8 * sizeof(int) + 16);
    for (size_t i = 0; i < c->n; ++i)
        fg[(size_t)((int)c->p[i].y - y0) * w + ((int)c->p[i].x - x0)] = 1;
    static const int k4[4][2] = {{1, 0}, {-1, 0}, {0, 1}, {0, -1}};
    int comps = 0, holes = 0;
    for (int pass = 0; pass < 3; ++pass) {
        /* pass 0: 8-connected fg components; 1: outer background from (0,0);
         * 2: remaining background components (holes) */
        for (int y = 0; y < h; ++y) {
            for (int x = 0; x < w; ++x) {
                const size_t at = (size_t)y * w + x;
                if (pass == 1 && (x || y)) continue;
                if (pass == 0 ? (!fg[at] || mark[at]) : (fg[at] || mark[at])) continue;
                if (pass == 0) ++comps;
                if (pass == 2) ++holes;
                size_t sp = 0;
                st[sp++] = x;
                st[sp++] = y;
                mark[at] = pass + 1;
                while (sp) {
                    const int cy = st[--sp], cx = st[--sp];
                    const int nk = pass == 0 ? 8 : 4;
                    for (int k = 0; k < nk; ++k) {
                        const int nx = cx + (pass == 0 ? kRing[k][0] : k4[k][0]);
                        const int ny = cy + (pass == 0 ? kRing[k][1] : k4[k][1]);
                        if (nx < 0 || nx >= w || ny < 0 || ny >= h) continue;
                        const size_t nat = (size_t)ny * w + nx;
                        if ((pass == 0 ? fg[nat] : !fg[nat]) && !mark[nat]) {
                            mark[nat] = pass + 1;
                            st[sp++] = nx;
                            st[sp++] = ny;
                        }
                    }
                }
            }
        }
    }
    free(fg);
    free(mark);
    free(st);
    return comps - holes;
}

/* shape_features (shape_features.cpp:147-251) + shape_feature_values order:
 * area, perimeter, bbox x/y/w/h, centroid x/y, circularity, extent,
 * aspect_ratio, convex_area, solidity, equivalent_diameter, major/minor axis,
 * eccentricity, elongation, orientation, euler_number, feret max/min, then the
 * 8 extrema as (x, y) pairs in regionprops order. */
static int shape_group(const cloud_t* c, double* o) {
    const double PI = 3.141592653589793, SQRT2 = 1.4142135623730951;
    memset(o, 0, 38 * sizeof(double));
    const size_t n = c->n;
    if (n == 0) return 0;
    const double dn = (double)n;
    const double bw = (double)((int)(c->bb.xmax - c->bb.xmin) + 1);
    const double bh = (double)((int)(c->bb.ymax - c->bb.ymin) + 1);
    o[0] = dn;
    o[2] = c->bb.xmin;
    o[3] = c->bb.ymin;
    o[4] = bw;
    o[5] = bh;
    o[9] = dn / (bw * bh);
    o[10] = bw / bh;
    double sx = 0, sy = 0;
    for (size_t i = 0; i < n; ++i) {
        sx += c->p[i].x;
        sy += c->p[i].y;
    }
    const double cx = sx / dn, cy = sy / dn;
    o[6] = cx;
    o[7] = cy;
    if (n == 1) {
        o[1] = 4.0;
        o[8] = 1.0;
    } else {  /* contour_perimeter (shape_features.cpp:11-21) over the traced cycle */
        int32_t* pts = NULL;
        size_t np = 0;
        int rc = trace_contour(c, &pts, &np);
        if (rc) return rc;
        double per = 4.0;
        if (np >= 2) {
            per = 0;
            for (size_t i = 0; i < np; ++i) {
                const size_t j = (i + 1) % np;
                const int dx = abs(pts[2 * i] - pts[2 * j]), dy = abs(pts[2 * i + 1] - pts[2 * j + 1]);
                per += (dx + dy == 2) ? SQRT2 : 1.0;
            }
        }
        free(pts);
        o[1] = per;
        o[8] = 4.0 * PI * dn / (per * per);
    }
    pt_t* hv = NULL;
    size_t nv = 0;
    if (convex_hull(c, &hv, &nv)) return 8;
    double carea = 0;  /* rasterized_hull_area (shape_features.cpp:102-115) */
    if (nv >= 3) {
        long long cnt = 0;
        for (int y = (int)c->bb.ymin; y <= (int)c->bb.ymax; ++y)
            for (int x = (int)c->bb.xmin; x <= (int)c->bb.xmax; ++x)
                if (point_in_hull(hv, nv, x, y)) ++cnt;
        carea = (double)cnt;
    }
    o[11] = carea;
    o[12] = carea > 0 ? dn / carea : 0.0;
    o[13] = sqrt(4.0 * dn / PI);
    {  /* +1/12 second-moment ellipse (shape_features.cpp:176-197), pixel order */
        double m20 = 0, m02 = 0, m11 = 0;
        for (size_t i = 0; i < n; ++i) {
            const double dx = c->p[i].x - cx, dy = c->p[i].y - cy;
            m20 += dx * dx;
            m02 += dy * dy;
            m11 += dx * dy;
        }
        const double a = m20 / dn + 1.0 / 12.0, cc = m02 / dn + 1.0 / 12.0, b = m11 / dn;
        const double disc = sqrt((a - cc) * (a - cc) / 4.0 + b * b);
        const double l1 = (a + cc) / 2.0 + disc, l2 = (a + cc) / 2.0 - disc;
        o[14] = 4.0 * sqrt(l1 > 0 ? l1 : 0.0);
        o[15] = 4.0 * sqrt(l2 > 0 ? l2 : 0.0);
        o[16] = l1 > 0 ? sqrt(fmax(0.0, 1.0 - l2 / l1)) : 0.0;
        o[17] = o[15] > 0 ? o[14] / o[15] : 0.0;
        double th = 0.5 * atan2(2.0 * b, a - cc);
        if (th <= -PI / 2.0) th += PI;
        o[18] = th;
    }
    o[19] = (double)euler_number(c);
    {  /* feret_diameters (shape_features.cpp:117-143) */
        double fmaxd = 0, fmind = 0;
        if (nv >= 2) {
            for (size_t i = 0; i < nv; ++i)
                for (size_t j = i + 1; j < nv; ++j)
                    fmaxd = fmax(fmaxd, hypot((double)(hv[i].x - hv[j].x), (double)(hv[i].y - hv[j].y)));
            if (nv > 2) {
                fmind = 1.79769313486231570815e308;
                for (size_t i = 0; i < nv; ++i) {
                    const pt_t a = hv[i], b = hv[(i + 1) % nv];
                    const double ex = b.x - a.x, ey = b.y - a.y, len = hypot(ex, ey);
                    double wd = 0;
                    for (size_t k = 0; k < nv; ++k) {
                        const double d = fabs(ex * (hv[k].y - a.y) - ey * (hv[k].x - a.x)) / len;
                        wd = fmax(wd, d);
                    }
                    fmind = fmin(fmind, wd);
                }
            }
        }
        o[20] = fmaxd;
        o[21] = fmind;
    }
    free(hv);
    {  /* extrema (shape_features.cpp:202-238) */
        int top = 1 << 30, bot = -1, left = 1 << 30, right = -1;
        for (size_t i = 0; i < n; ++i) {
            const int x = (int)c->p[i].x, y = (int)c->p[i].y;
            top = y < top ? y : top;
            bot = y > bot ? y : bot;
            left = x < left ? x : left;
            right = x > right ? x : right;
        }
        int tl = 1 << 30, tr = -1, bl = 1 << 30, br = -1, lt = 1 << 30, lb = -1, rt = 1 << 30, rb = -1;
        for (size_t i = 0; i < n; ++i) {
            const int x = (int)c->p[i].x, y = (int)c->p[i].y;
            if (y == top) { tl = x < tl ? x : tl; tr = x > tr ? x : tr; }
            if (y == bot) { bl = x < bl ? x : bl; br = x > br ? x : br; }
            if (x == left) { lt = y < lt ? y : lt; lb = y > lb ? y : lb; }
            if (x == right) { rt = y < rt ? y : rt; rb = y > rb ? y : rb; }
        }
        const int ex[8] = {tl, tr, right, right, br, bl, left, left};
        const int ey[8] = {top, top, rt, rb, bot, bot, lb, lt};
        for (int i = 0; i < 8; ++i) {
            o[22 + 2 * i] = ex[i];
            o[23 + 2 * i] = ey[i];
        }
    }
    return 0;
}

/* ------------------------------------------------------------- dispatch -- */

static int check_groups(unsigned groups) {
    if (groups == 0) return fail(1, "feature list is empty");
    return 0;
}

/* compute_roi_features (engine.cpp:138-209), all seven groups. */
static int roi_features(const cloud_t* c, unsigned groups, const fxo_params* prm, double* out) {
    double* o = out;
    int rc;
    if (groups & FXO_INTENSITY) {
        if ((rc = intensity_group(c, prm->histogram_bins, o))) return rc;
        o += 39;
    }
    if (groups & FXO_SHAPE) {
        if ((rc = shape_group(c, o))) return rc;
        o += 38;
    }
    if (groups & FXO_MOMENTS) {
        moments_t b, w;
        compute_moments(c, 0, &b);
        if (compute_moments(c, 1, &w) == 6) memset(&w, 0, sizeof w); /* engine.cpp:184-188 */
        o = append_moments(&b, o);
        o = append_moments(&w, o);
    }
    if (groups & FXO_GLCM) {
        if ((rc = glcm_group(c, prm, o))) return rc;
        o += 29 * (prm->n_angles + 1);
    }
    if (groups & (FXO_GLRLM | FXO_GLSZM | FXO_NGTDM)) {
        if ((rc = rlzn_groups(c, groups, prm, &o))) return rc;
    }
    return 0;
}

static void cloud_bbox(cloud_t* c) {
    if (!c->n) return;
    c->bb.xmin = c->bb.xmax = c->p[0].x;
    c->bb.ymin = c->bb.ymax = c->p[0].y;
    for (size_t i = 0; i < c->n; ++i) {
        if (c->p[i].x < c->bb.xmin) c->bb.xmin = c->p[i].x;
        if (c->p[i].x > c->bb.xmax) c->bb.xmax = c->p[i].x;
        if (c->p[i].y < c->bb.ymin) c->bb.ymin = c->p[i].y;
        if (c->p[i].y > c->bb.ymax) c->bb.ymax = c->p[i].y;
    }
}

int fxo_roi_features(const uint32_t* xs, const uint32_t* ys, const uint16_t* is, size_t n,
                     unsigned groups, const fxo_params* p, double* out, size_t cap,
                     int* n_cols) {
    int rc = check_groups(groups);
    if (rc) return rc;
    *n_cols = fxo_n_cols(groups, p);
    if ((size_t)*n_cols > cap) return fail(10, "capacity");
    px_t* px = malloc((n ? n : 1) * sizeof(px_t));
    for (size_t i = 0; i < n; ++i) px[i] = (px_t){xs[i], ys[i], is[i]};
    cloud_t c = {px, n, {0, 0, 0, 0}};
    cloud_bbox(&c);
    rc = roi_features(&c, groups, p, out);
    free(px);
    return rc;
}

int fxo_featurize(const uint16_t* intensity, const uint16_t* labels, int w, int h,
                  unsigned groups, const fxo_params* p, uint32_t* out_labels,
                  double* out_values, size_t cap_rois, size_t* n_rois, int* n_cols) {
    int rc = check_groups(groups);
    if (rc) return rc;
    const int nc = fxo_n_cols(groups, p);
    *n_cols = nc;
    const size_t npx = (size_t)w * h;
    /* gather clouds in mask scan order (roi.cpp:82-105) by a counting sort */
    size_t* start = calloc(65537, sizeof(size_t));
    for (size_t i = 0; i < npx; ++i)
        if (labels[i]) start[labels[i] + 1]++;
    size_t k = 0;
    for (int l = 1; l < 65536; ++l)
        if (start[l + 1]) ++k;
    *n_rois = k;
    if (k > cap_rois) {
        free(start);
        return fail(10, "capacity");
    }
    for (int l = 1; l <= 65536; ++l) start[l] += start[l - 1];
    size_t fg = start[65536];
    px_t* all = malloc((fg ? fg : 1) * sizeof(px_t));
    size_t* cur = malloc(65537 * sizeof(size_t));
    memcpy(cur, start, 65537 * sizeof(size_t));
    for (size_t i = 0; i < npx; ++i) {
        const uint16_t l = labels[i];
        if (!l) continue;
        all[cur[l]++] = (px_t){(uint32_t)(i % (size_t)w), (uint32_t)(i / (size_t)w), intensity[i]};
    }
    size_t r = 0;
    for (int l = 1; l < 65536 && !rc; ++l) {
        const size_t cnt = start[l + 1] - start[l];
        if (!cnt) continue;
        cloud_t c = {all + start[l], cnt, {0, 0, 0, 0}};
        cloud_bbox(&c);
        out_labels[r] = (uint32_t)l;
        rc = roi_features(&c, groups, p, out_values + r * (size_t)nc);
        ++r;
    }
    free(all);
    free(cur);
    free(start);
    return rc;
}

int fxo_trace_contour(const uint32_t* xs, const uint32_t* ys, size_t n, int32_t* out_xy,
                      size_t cap, size_t* n_points) {
    px_t* px = malloc((n ? n : 1) * sizeof(px_t));
    for (size_t i = 0; i < n; ++i) px[i] = (px_t){xs[i], ys[i], 1};
    cloud_t c = {px, n, {0, 0, 0, 0}};
    cloud_bbox(&c);
    int32_t* pts = NULL;
    int rc = trace_contour(&c, &pts, n_points);
    if (!rc && *n_points <= cap) memcpy(out_xy, pts, *n_points * 2 * sizeof(int32_t));
    if (!rc && *n_points > cap) rc = fail(10, "capacity");
    free(pts);
    free(px);
    return rc;
}

int fxo_glcm_counts(const uint32_t* xs, const uint32_t* ys, const uint16_t* is, size_t n,
                    int ng, int offset, int angle, int symmetric, uint64_t* counts,
                    uint64_t* pair_count) {
    px_t* px = malloc((n ? n : 1) * sizeof(px_t));
    for (size_t i = 0; i < n; ++i) px[i] = (px_t){xs[i], ys[i], is[i]};
    cloud_t c = {px, n, {0, 0, 0, 0}};
    cloud_bbox(&c);
    droi_t r;
    memset(&r, 0, sizeof r);
    int rc = discretize(&c, ng, &r);
    if (!rc) rc = glcm_count(&r, offset, angle, symmetric, counts, pair_count);
    free(r.grid);
    free(px);
    return rc;
}

/* histogram of intensity_features.cpp:156-167 */
int fxo_intensity_hist(const uint16_t* is, size_t n, int bins, uint64_t* hist) {
    const int nb = bins > 2 ? bins : 2;
    memset(hist, 0, (size_t)nb * sizeof(uint64_t));
    if (!n) return 0;
    double mn = is[0], mx = is[0];
    for (size_t i = 0; i < n; ++i) {
        if (is[i] < mn) mn = is[i];
        if (is[i] > mx) mx = is[i];
    }
    const double range = mx - mn;
    if (range == 0) {
        hist[0] = n;
        return 0;
    }
    for (size_t i = 0; i < n; ++i) {
        int b = (int)((double)nb * ((double)is[i] - mn) / range);
        if (b >= nb) b = nb - 1;
        ++hist[b];
    }
    return 0;
}
