/*
 * oracle.c -- CPU restatement of the reference (pyrocell 0.1.0) wildfire CA
 * path.  TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs as the checker and the
 * CPU baseline.  Nothing in the product package links or calls this file.
 *
 * Every function restates the reference algorithm in plain fp64 C; the
 * reference file:line each piece follows is cited next to it (paths relative
 * to the reference's pkg/src/pyrocell/).  The restatement is pinned by the
 * reference's own golden vectors (tests/test_rng.py:7-23) and by fixtures
 * produced by running the reference itself (tests/golden/make_golden.py).
 *
 * Threading: an OpenMP row partition of the active window, the analogue of
 * kernel.py:307-327's row bands.  Draws are keyed per absolute cell
 * (rng.py:55-75), so any partition gives bit-identical results.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------- RNG --- */
/* rng.py:19-21 constants; rng.py:35-39 finalizer. */
#define ORC_GOLDEN 0x9E3779B97F4A7C15ULL

static inline uint64_t orc_mix(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* rng.py:46-52: per-(seed, step, channel) stream key. */
uint64_t orc_stream_key(uint64_t seed, uint64_t t, uint64_t channel) {
    uint64_t k = orc_mix(seed + ORC_GOLDEN);
    k ^= t * 0x9E3779B97F4A7C16ULL;
    k ^= channel * 0xD1B54A32D192ED03ULL;
    return orc_mix(k);
}

/* rng.py:70-75: fold the absolute cell into the key, keep the top 53 bits. */
static inline double orc_cell_draw(uint64_t key, uint64_t row, uint64_t col) {
    uint64_t code = (row << 32) | col;
    uint64_t mixed = orc_mix(orc_mix(code + ORC_GOLDEN) ^ key);
    return (double)(mixed >> 11) * 0x1p-53;
}

/* rng.py:55-75 uniform_grid. */
void orc_uniform_grid(uint64_t seed, uint64_t t, uint64_t channel, int64_t row0,
                      int64_t col0, int64_t height, int64_t width, double* out) {
    uint64_t key = orc_stream_key(seed, t, channel);
    for (int64_t i = 0; i < height; ++i)
        for (int64_t j = 0; j < width; ++j)
            out[i * width + j] = orc_cell_draw(key, (uint64_t)(row0 + i), (uint64_t)(col0 + j));
}

/* rng.py:83-88 derive_epoch_seed. */
uint64_t orc_epoch_seed(uint64_t base_seed, uint64_t epoch) {
    uint64_t k = orc_mix(base_seed + ORC_GOLDEN);
    k ^= epoch * 0xD1342543DE82EF95ULL;
    return orc_mix(k);
}

/* ------------------------------------------------------------- slope --- */
/* data_io.py:92-132 slope_from_altitude: out is (h, w, 3, 3) degrees;
 * each forward pair computed once and negated for the mirror entry. */
int orc_slope_from_altitude(const double* e, int h, int w, double cell_side,
                            int uphill_positive, double* out) {
    if (cell_side <= 0) return -1;
    memset(out, 0, sizeof(double) * (size_t)h * w * 9);
    static const int fwd[4][2] = {{0, 1}, {1, -1}, {1, 0}, {1, 1}};
    const double rad2deg = 180.0 / 3.141592653589793;
    for (int f = 0; f < 4; ++f) {
        int dr = fwd[f][0], dc = fwd[f][1];
        double k = (dr != 0 && dc != 0) ? sqrt(2.0) : 1.0;
        double denom = k * cell_side;
        for (int r = 0; r < h; ++r) {
            int r2 = r + dr;
            if (r2 < 0 || r2 >= h) continue;
            for (int c = 0; c < w; ++c) {
                int c2 = c + dc;
                if (c2 < 0 || c2 >= w) continue;
                double th = atan((e[(size_t)r * w + c] - e[(size_t)r2 * w + c2]) / denom) * rad2deg;
                out[((size_t)r * w + c) * 9 + (1 + dr) * 3 + (1 + dc)] = th;
                out[((size_t)r2 * w + c2) * 9 + (1 - dr) * 3 + (1 - dc)] = -th;
            }
        }
    }
    if (uphill_positive)
        for (size_t i = 0; i < (size_t)h * w * 9; ++i) out[i] = -out[i];
    return 0;
}

/* --------------------------------------------------------- CA kernel --- */
/* kernel.py:30-34 slot order NW,N,NE,W,E,SW,S,SE (neighbour position
 * relative to the target); kernel.py:38-47 bearing of the propagation
 * direction arriving from each slot. */
static const int ORC_POS[8][2] = {{-1, -1}, {-1, 0}, {-1, 1}, {0, -1},
                                  {0, 1},   {1, -1}, {1, 0},  {1, 1}};
static const double ORC_BEAR[8] = {315.0, 270.0, 225.0, 0.0, 180.0, 45.0, 90.0, 135.0};

typedef struct {
    int h, w;
    const double* vw;      /* (h,w) wind speed                       */
    const double* wdir;    /* (h,w) wind direction, deg East-CCW     */
    const double* slope9;  /* (h,w,3,3) slope toward neighbour, deg  */
    const double* canopy;  /* (h,w)                                  */
    const double* density; /* (h,w)                                  */
    double c1, c2, a, p_h, p_continue, norm_c;
    int factor_source;     /* 0 = "target" (default), 1 = "source"   */
    int slope_radians;     /* slope_units == "radians"               */
    int64_t row0, col0;    /* absolute position of local cell (0, 0): draws are keyed
                              by the absolute cell (rng.py:64-67), so a crop of a
                              larger domain sees the domain's draws               */
    const double* wsched;  /* NULL, or [steps][4] per pre-step index t: the wind of
                              step t is a WindUpdate (kernel.py:422-428) with fields
                              alpha*V + beta and theta + gamma (base fields vw/wdir) */
} orc_model;

/* One slot's cached quantities, restating build_fields (kernel.py:165-195)
 * for a single (source cell, slot) pair. */
typedef struct { double fp, raw, rest, vw, cosm1, slope; } orc_slot;

static inline void orc_slot_eval(const orc_model* m, const double* vw, const double* wdir,
                                 const double* ws, int sr, int sc, int tr, int tc, int k,
                                 orc_slot* o) {
    const int w = m->w;
    size_t src = (size_t)sr * w + sc, tgt = (size_t)tr * w + tc;
    int dr = -ORC_POS[k][0], dc = -ORC_POS[k][1];
    double v = vw[src], th = wdir[src];
    if (ws) {  /* the WindUpdate's fields, computed elementwise in fp64 */
        v = ws[0] * v + ws[1];
        th = th + ws[2];
    }
    double cosm1 = cos((th - ORC_BEAR[k]) * (3.141592653589793 / 180.0)) - 1.0;
    double s = m->slope9[src * 9 + (1 + dr) * 3 + (1 + dc)];
    if (m->slope_radians) s = s * (180.0 / 3.141592653589793);
    size_t site = m->factor_source ? src : tgt;
    double vd = (1.0 + m->canopy[site]) * (1.0 + m->density[site]);   /* kernel.py:172-174 */
    double exp_c1 = exp(m->c1 * v);                                    /* kernel.py:175 */
    double rest = vd * exp_c1 * exp(m->c2 * v * cosm1) * exp(m->a * s); /* kernel.py:188 */
    double raw = m->p_h * rest;                                        /* kernel.py:189 */
    o->fp = tanh(m->norm_c * raw);                                     /* kernel.py:190 */
    o->raw = raw; o->rest = rest; o->vw = v; o->cosm1 = cosm1; o->slope = s;
}

/* Conditioning of J for an fp32 evaluation of the same formulas (test
 * infrastructure: the scale against which an fp32 J is judged).  A slot's
 * exponent c1 V + c2 V (cos - 1) + a S carries an absolute error of about
 * E 2^-23 with E = |c1 V| + |c2| (|V (cos - 1)| + 4 |V|) + |a S| (fp32
 * operands; the wind term is formed from an fp32 wind vector), so its factor
 * 1 - fp has relative error r = 2^-23 (E + 2) (1 + 2y) once y = c raw
 * saturates (1 - tanh y ~ 2 e^-2y amplifies the error of y by 2y).  Each
 * term of J is a product over the live slots' factors: its bound is the term
 * times the sum of r; the c2 term adds the absolute error of cos - 1 formed
 * from the fp32 wind vector, 2^-21 |chain raw V|. */
static void orc_fp32_cond(const orc_model* m, const orc_slot* sl, const int* live,
                          const double* pre, const double* suf, double* out) {
    double R = 0.0;
    for (int k = 0; k < 8; ++k) {
        if (!live[k]) continue;
        const double v = fabs(sl[k].vw);
        const double E = fabs(m->c1) * v + fabs(m->c2) * (v * fabs(sl[k].cosm1) + 4.0 * v) +
                         fabs(m->a * sl[k].slope);
        const double y = m->norm_c * sl[k].raw;
        R += 0x1p-23 * (E + 2.0) * (1.0 + (y > 0.55 ? 2.0 * y : 0.0));
    }
    double o0 = 0, o1 = 0, o2 = 0, o3 = 0;
    for (int k = 0; k < 8; ++k) {
        if (!live[k]) continue;
        const double ch = fabs(pre[k] * suf[k] * (m->norm_c * (1.0 - sl[k].fp * sl[k].fp)));
        o0 += ch * fabs(sl[k].raw * sl[k].vw) * R;
        o1 += ch * fabs(sl[k].raw * sl[k].vw) * (fabs(sl[k].cosm1) * R + 0x1p-21);
        o2 += ch * fabs(sl[k].raw * sl[k].slope) * R;
        o3 += ch * fabs(sl[k].rest) * R;
    }
    out[0] = o0; out[1] = o1; out[2] = o2; out[3] = o3;
}

/* Precomputed per-slot normalized probabilities, fp[k][i] at source cell i
 * (the fields of build_fields, kernel.py:177-190). */
static void orc_build_fp(const orc_model* m, const double* vw, const double* wdir, double* fp) {
    const int h = m->h, w = m->w;
#pragma omp parallel for schedule(static)
    for (int r = 0; r < h; ++r) {
        for (int c = 0; c < w; ++c) {
            for (int k = 0; k < 8; ++k) {
                int tr = r - ORC_POS[k][0], tc = c - ORC_POS[k][1];
                double val = 0.0;
                if (tr >= 0 && tr < h && tc >= 0 && tc < w) {
                    orc_slot s;
                    orc_slot_eval(m, vw, wdir, NULL, r, c, tr, tc, k, &s);
                    val = s.fp;
                } else {
                    /* target outside the grid: the reference still fills the
                     * field (vd of the zero-padded shift); never consumed. */
                    val = 0.0;
                }
                fp[(size_t)k * h * w + (size_t)r * w + c] = val;
            }
        }
    }
}

/*
 * orc_run -- restates run_simulation (kernel.py:453-529) with step_forward
 * (kernel.py:263-333), _step_band (kernel.py:216-256) and the tape
 * recording (kernel.py:336-402) folded into a per-cell Jacobian
 * J_j = sum_k chain_k / g  (tape.py:134-147 with g factored out).
 *
 * wind schedule: n_wind updates, wind_at[i] = 1-based step, fields
 * wind_v/wind_d [n_wind][h][w] (kernel.py:505-511: applied before the step).
 * attach: array of steps+1 flags, attach[s] for 1-based step s.
 * Outputs: burning/burned (uint8), acc (fp64), t_ign (int32: pre-step index
 * of ignition, -1 initial, INT32_MAX never), jac (h*w*4 fp64, may be NULL),
 * jac_abs (h*w*4: the sum of the absolute slot terms of each J component --
 * the scale against which a rounded J is judged; may be NULL), jac_floor
 * (h*w*4: the absolute rounding floor of the reference's own J -- where a
 * slot saturates, fp is within ulps of 1 and the factors 1 - fp and 1 - fp^2
 * of tape.py:106-147 cancel; each term recomputed with those factors
 * inflated by their fp64 error, minus the term; may be NULL), jac_cond
 * (h*w*4: the fp32 conditioning of J -- see orc_fp32_cond; may be NULL),
 * series (steps*2 int64: burning, burned after each step),
 * n_entries (tape entries = ignitions on attached steps).
 */
int orc_run(const orc_model* m, const uint8_t* init, int steps, uint64_t seed,
            int n_wind, const int* wind_at, const double* wind_v, const double* wind_d,
            const uint8_t* attach, int threads,
            uint8_t* burning, uint8_t* burned, double* acc, int32_t* t_ign,
            double* jac, double* jac_abs, double* jac_floor, double* jac_cond,
            int64_t* series, int64_t* n_entries) {
    const int h = m->h, w = m->w;
    const size_t n = (size_t)h * w;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#else
    (void)threads;
#endif
    if (steps < 0) return -1;
    /* new_fire_state, model.py:180-200 */
    int64_t nburning = 0;
    for (size_t i = 0; i < n; ++i) {
        burning[i] = init[i] ? 1 : 0;
        burned[i] = 0;
        acc[i] = init[i] ? 1.0 : 0.0;
        t_ign[i] = init[i] ? -1 : INT32_MAX;
        nburning += burning[i];
    }
    if (jac) memset(jac, 0, sizeof(double) * n * 4);
    if (jac_abs) memset(jac_abs, 0, sizeof(double) * n * 4);
    if (jac_floor) memset(jac_floor, 0, sizeof(double) * n * 4);
    if (jac_cond) memset(jac_cond, 0, sizeof(double) * n * 4);
    int64_t nburned = 0, entries = 0;

    double* fp = (double*)malloc(sizeof(double) * n * 8);
    uint8_t* prev = (uint8_t*)malloc(n);
    if (!fp || !prev) { free(fp); free(prev); return -2; }
    const double* vw = m->vw;
    const double* wdir = m->wdir;
    if (!m->wsched) orc_build_fp(m, vw, wdir, fp);
    int next_wind = 0;

    for (int s = 1; s <= steps; ++s) {
        while (next_wind < n_wind && wind_at[next_wind] == s) {   /* kernel.py:505-511 */
            vw = wind_v + (size_t)next_wind * n;
            wdir = wind_d + (size_t)next_wind * n;
            if (!m->wsched) orc_build_fp(m, vw, wdir, fp);
            ++next_wind;
        }
        const uint64_t t = (uint64_t)(s - 1);  /* pre-step index, kernel.py:295 */
        /* parametric schedule: the step's fields are evaluated per live slot
         * (the same values build_fields would tabulate for this step) */
        const double* ws = m->wsched ? m->wsched + (size_t)t * 4 : NULL;
        int do_attach = attach ? attach[s] : 0;
        /* _burning_bbox, kernel.py:208-213, + 1-cell margin kernel.py:301-302 */
        int rmin = h, rmax = -1, cmin = w, cmax = -1;
        for (int r = 0; r < h; ++r) {
            const uint8_t* row = burning + (size_t)r * w;
            for (int c = 0; c < w; ++c)
                if (row[c]) {
                    if (r < rmin) rmin = r;
                    if (r > rmax) rmax = r;
                    if (c < cmin) cmin = c;
                    if (c > cmax) cmax = c;
                }
        }
        if (rmax >= 0) {
            int r0 = rmin > 0 ? rmin - 1 : 0, r1 = rmax + 2 < h ? rmax + 2 : h;
            int c0 = cmin > 0 ? cmin - 1 : 0, c1 = cmax + 2 < w ? cmax + 2 : w;
            /* prev_burning copy, kernel.py:304-305 (only rows that can hold fire) */
            memcpy(prev + (size_t)rmin * w, burning + (size_t)rmin * w, (size_t)(rmax - rmin + 1) * w);
            /* rows the window's neighbours can read but that hold no fire */
            for (int r = (rmin >= 2 ? rmin - 2 : 0); r < rmin; ++r) memset(prev + (size_t)r * w, 0, w);
            for (int r = rmax + 1; r < (rmax + 3 < h ? rmax + 3 : h); ++r) memset(prev + (size_t)r * w, 0, w);
            const uint64_t key_i = orc_stream_key(seed, t, 0);
            const uint64_t key_c = orc_stream_key(seed, t, 1);
            int64_t d_ign = 0, d_out = 0, d_ent = 0;
#pragma omp parallel for schedule(static) reduction(+ : d_ign, d_out, d_ent)
            for (int r = r0; r < r1; ++r) {
                for (int c = c0; c < c1; ++c) {
                    size_t j = (size_t)r * w + c;
                    if (prev[j]) {
                        /* keeps = burning & (u_C < p_continue), kernel.py:248-253 */
                        double u = orc_cell_draw(key_c, (uint64_t)(r + m->row0),
                                                 (uint64_t)(c + m->col0));
                        if (!(u < m->p_continue)) {
                            burning[j] = 0;
                            burned[j] = 1;
                            ++d_out;
                        }
                        continue;
                    }
                    if (burned[j]) continue;
                    /* p = 1 - prod_k (1 - fp_k * B), slot order, kernel.py:232-240 */
                    double prod = 1.0;
                    int any = 0;
                    for (int k = 0; k < 8; ++k) {
                        int sr = r + ORC_POS[k][0], sc = c + ORC_POS[k][1];
                        if (sr < 0 || sr >= h || sc < 0 || sc >= w) continue;
                        size_t i = (size_t)sr * w + sc;
                        if (!prev[i]) continue;
                        double f;
                        if (ws) {
                            orc_slot sk;
                            orc_slot_eval(m, vw, wdir, ws, sr, sc, r, c, k, &sk);
                            f = sk.fp;
                        } else {
                            f = fp[(size_t)k * n + i];
                        }
                        prod *= 1.0 - f;
                        any = 1;
                    }
                    if (!any) continue;
                    double p = 1.0 - prod;
                    double u = orc_cell_draw(key_i, (uint64_t)(r + m->row0), (uint64_t)(c + m->col0));
                    if (!(u < p)) continue;  /* kernel.py:246-247 strict < */
                    burning[j] = 1;
                    acc[j] = p;              /* kernel.py:254-255 */
                    t_ign[j] = (int32_t)t;
                    ++d_ign;
                    if (do_attach && jac) {
                        /* tape.py:134-147: chain_k = g * prod_{m!=k}(1-f_m) * c(1-f_k^2) */
                        orc_slot sl[8];
                        double fac[8];
                        int live[8];
                        for (int k = 0; k < 8; ++k) {
                            int sr = r + ORC_POS[k][0], sc = c + ORC_POS[k][1];
                            live[k] = (sr >= 0 && sr < h && sc >= 0 && sc < w &&
                                       prev[(size_t)sr * w + sc]);
                            if (live[k]) {
                                orc_slot_eval(m, vw, wdir, ws, sr, sc, r, c, k, &sl[k]);
                                fac[k] = 1.0 - sl[k].fp;
                            } else {
                                fac[k] = 1.0;
                            }
                        }
                        double pre[8], suf[8];  /* tape.py:106-115 leave-one-out */
                        pre[0] = 1.0;
                        suf[7] = 1.0;
                        for (int k = 1; k < 8; ++k) {
                            pre[k] = pre[k - 1] * fac[k - 1];
                            suf[7 - k] = suf[8 - k] * fac[8 - k];
                        }
                        double g0 = 0, g1 = 0, g2 = 0, g3 = 0;
                        double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
                        double f0 = 0, f1 = 0, f2 = 0, f3 = 0;
                        /* rounding floor: every factor that cancels near a
                         * saturated slot (1 - fp, 1 - fp^2 with fp within ulps
                         * of 1) inflated by its fp64 absolute error (a tanh
                         * within 2 ulps on either side: 2^-50, and 2^-49 for
                         * the square) -- an interval bound on |J - J_exact| */
                        double hp[8], hs[8];
                        hp[0] = 1.0;
                        hs[7] = 1.0;
                        for (int k = 1; k < 8; ++k) {
                            hp[k] = hp[k - 1] * (live[k - 1] ? fac[k - 1] + 0x1p-50 : 1.0);
                            hs[7 - k] = hs[8 - k] * (live[8 - k] ? fac[8 - k] + 0x1p-50 : 1.0);
                        }
                        for (int k = 0; k < 8; ++k) {
                            if (!live[k]) continue;
                            double ch = pre[k] * suf[k] * (m->norm_c * (1.0 - sl[k].fp * sl[k].fp));
                            double t0_ = ch * sl[k].raw * sl[k].vw;
                            double t1_ = ch * sl[k].raw * sl[k].vw * sl[k].cosm1;
                            double t2_ = ch * sl[k].raw * sl[k].slope;
                            double t3_ = ch * sl[k].rest;
                            g0 += t0_; g1 += t1_; g2 += t2_; g3 += t3_;
                            a0 += fabs(t0_); a1 += fabs(t1_); a2 += fabs(t2_); a3 += fabs(t3_);
                            double chh = hp[k] * hs[k] *
                                         (m->norm_c * (fabs(1.0 - sl[k].fp * sl[k].fp) + 0x1p-49));
                            f0 += fabs(chh * sl[k].raw * sl[k].vw) - fabs(t0_);
                            f1 += fabs(chh * sl[k].raw * sl[k].vw * sl[k].cosm1) - fabs(t1_);
                            f2 += fabs(chh * sl[k].raw * sl[k].slope) - fabs(t2_);
                            f3 += fabs(chh * sl[k].rest) - fabs(t3_);
                        }
                        if (jac_abs) {
                            jac_abs[j * 4 + 0] = a0; jac_abs[j * 4 + 1] = a1;
                            jac_abs[j * 4 + 2] = a2; jac_abs[j * 4 + 3] = a3;
                        }
                        if (jac_floor) {
                            jac_floor[j * 4 + 0] = f0; jac_floor[j * 4 + 1] = f1;
                            jac_floor[j * 4 + 2] = f2; jac_floor[j * 4 + 3] = f3;
                        }
                        if (jac_cond) orc_fp32_cond(m, sl, live, pre, suf, jac_cond + j * 4);
                        jac[j * 4 + 0] = g0;
                        jac[j * 4 + 1] = g1;
                        jac[j * 4 + 2] = g2;
                        jac[j * 4 + 3] = g3;
                        ++d_ent;
                    }
                }
            }
            nburning += d_ign - d_out;
            nburned += d_out;
            entries += d_ent;
        }
        if (series) {   /* kernel.py:518-522 per-step counts */
            series[(size_t)(s - 1) * 2 + 0] = nburning;
            series[(size_t)(s - 1) * 2 + 1] = nburned;
        }
    }
    free(fp);
    free(prev);
    if (n_entries) *n_entries = entries;
    return 0;
}

/* -------------------------------------------------------------- loss --- */
/* losses.py:32-86 combined_loss: union-bbox BCE-with-logits mean + MSE of
 * 4x4 average pools (remainder truncated), plus the exact dL/dacc. */
int orc_combined_loss(const double* acc, const uint8_t* target, int h, int w,
                      double* grad, double* terms /* bce, mse */, int* crop /* r0,r1,c0,c1 */) {
    int r0 = h, r1 = -1, c0 = w, c1 = -1;
    for (int r = 0; r < h; ++r)
        for (int c = 0; c < w; ++c) {
            size_t i = (size_t)r * w + c;
            if (acc[i] != 0.0 || target[i]) {
                if (r < r0) r0 = r;
                if (r > r1) r1 = r;
                if (c < c0) c0 = c;
                if (c > c1) c1 = c;
            }
        }
    if (r1 < 0) { r0 = 0; r1 = h; c0 = 0; c1 = w; }   /* losses.py:23-28 */
    else { r1 += 1; c1 += 1; }
    double n_crop = (double)(r1 - r0) * (double)(c1 - c0);
    double bce = 0.0;
    if (grad) memset(grad, 0, sizeof(double) * (size_t)h * w);
    for (int r = r0; r < r1; ++r)
        for (int c = c0; c < c1; ++c) {
            size_t i = (size_t)r * w + c;
            double x = acc[i], y = target[i] ? 1.0 : 0.0;
            bce += (x > 0.0 ? x : 0.0) - x * y + log1p(exp(-fabs(x)));
            if (grad) {
                double sig = x >= 0 ? 1.0 / (1.0 + exp(-x)) : exp(x) / (1.0 + exp(x));
                grad[i] = (sig - y) / n_crop;
            }
        }
    bce /= n_crop;
    double mse = 0.0;
    int hp = h / 4, wp = w / 4;
    if (hp > 0 && wp > 0) {
        double npool = (double)hp * wp;
        for (int pr = 0; pr < hp; ++pr)
            for (int pc = 0; pc < wp; ++pc) {
                double sx = 0.0, sy = 0.0;
                for (int a = 0; a < 4; ++a)
                    for (int b = 0; b < 4; ++b) {
                        size_t i = (size_t)(pr * 4 + a) * w + pc * 4 + b;
                        sx += acc[i];
                        sy += target[i] ? 1.0 : 0.0;
                    }
                double diff = sy / 16.0 - sx / 16.0;
                mse += diff * diff;
                if (grad) {
                    double cg = -2.0 * diff / (16.0 * npool);
                    for (int a = 0; a < 4; ++a)
                        for (int b = 0; b < 4; ++b)
                            grad[(size_t)(pr * 4 + a) * w + pc * 4 + b] += cg;
                }
            }
        mse /= npool;
    }
    terms[0] = bce;
    terms[1] = mse;
    crop[0] = r0; crop[1] = r1; crop[2] = c0; crop[3] = c1;
    return 0;
}

/* tape.py:118-148 backward_params in the per-cell-Jacobian form:
 * grad = sum_j dL/dacc_j * J_j, returned as (c1, c2, a, p_h). */
void orc_contract(const double* jac, const double* g, int64_t n, double* out) {
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    for (int64_t i = 0; i < n; ++i) {
        double gi = g[i];
        if (gi == 0.0) continue;
        s0 += gi * jac[i * 4 + 0];
        s1 += gi * jac[i * 4 + 1];
        s2 += gi * jac[i * 4 + 2];
        s3 += gi * jac[i * 4 + 3];
    }
    out[0] = s0; out[1] = s1; out[2] = s2; out[3] = s3;
}
