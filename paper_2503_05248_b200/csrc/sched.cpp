// Host scheduler: Algorithm 1 (memory-constrained) with the
// chance-constrained bound of Eqs. 7-11 refreshing the safety
// buffer L0 (Eqs. 12-13), Algorithm 2 (SLA-constrained,
// PAPER.md:221-250), the min-combination and the static baseline
// (PAPER.md:71).  All decisions are integer-exact (R6, R11-R16).
#include <algorithm>
#include <cmath>
#include <deque>
#include <new>
#include <utility>

#include "common.h"

namespace {

using i128 = __int128;
constexpr int kThetaShift = 24;

// Wichura, AS241 (PPND16): standard normal quantile, |rel err| ~ 1e-16.
double normal_quantile(double p) {
    const double q = p - 0.5;
    if (std::fabs(q) <= 0.425) {
        const double r = 0.180625 - q * q;
        const double num = (((((((2.5090809287301226727e+3 * r + 3.3430575583588128105e+4) * r +
                                 6.7265770927008700853e+4) * r + 4.5921953931549871457e+4) * r +
                               1.3731693765509461125e+4) * r + 1.9715909503065514427e+3) * r +
                             1.3314166789178437745e+2) * r + 3.3871328727963666080e+0) * q;
        const double den = (((((((5.2264952788528545610e+3 * r + 2.8729085735721942674e+4) * r +
                                 3.9307895800092710610e+4) * r + 2.1213794301586595867e+4) * r +
                               5.3941960214247511077e+3) * r + 6.8718700749205790830e+2) * r +
                             4.2313330701600911252e+1) * r + 1.0);
        return num / den;
    }
    double r = q <= 0.0 ? p : 1.0 - p;
    r = std::sqrt(-std::log(r));
    double num, den;
    if (r <= 5.0) {
        r -= 1.6;
        num = (((((((7.7454501427834140764e-4 * r + 2.2723844989269184583e-2) * r +
                    2.4178072517745061177e-1) * r + 1.2704582524523683826e+0) * r +
                  3.6478483247632045605e+0) * r + 5.7694972214606914055e+0) * r +
                4.6303378461565452959e+0) * r + 1.4234371107496835773e+0);
        den = (((((((1.0507500716444168432e-9 * r + 5.4759380849953449460e-4) * r +
                    1.5198666563616457197e-2) * r + 1.4810397642748007459e-1) * r +
                  6.8976733498510000455e-1) * r + 1.6763848301838038494e+0) * r +
                2.0531916266377588219e+0) * r + 1.0);
    } else {
        r -= 5.0;
        num = (((((((2.0103343992922881327e-7 * r + 2.7115555687434875782e-5) * r +
                    1.2426609473880784386e-3) * r + 2.6532189526576123093e-2) * r +
                  2.9656057182850489123e-1) * r + 1.7848265399172913358e+0) * r +
                5.4637849111641143699e+0) * r + 6.6579046435011037772e+0);
        den = (((((((2.0442631033899397856e-15 * r + 1.4215117583164458887e-7) * r +
                    1.8463183175100546818e-5) * r + 7.8686913114561325910e-4) * r +
                  1.4875361290850614853e-2) * r + 1.3692988092273580531e-1) * r +
                5.9983220655588793769e-1) * r + 1.0);
    }
    const double x = num / den;
    return q < 0.0 ? -x : x;
}

// eta - b m >= theta sqrt(b v)  <=>  A = n eta - b S >= 0  and  A^2 2^48 >= tq^2 b V2   (R6)
bool feasible(int64_t b, int64_t n, int64_t S, int64_t V2, int64_t eta, int64_t tq) {
    const i128 A = static_cast<i128>(n) * eta - static_cast<i128>(b) * S;
    if (A < 0) return false;
    // A^2 * 2^48 may exceed int128 for huge windows; compare A^2 >= (tq^2 b V2) / 2^48 exactly
    const i128 lhs = A * A;
    const i128 t2 = static_cast<i128>(tq) * tq;          // < 2^60
    const i128 rhs_num = t2 * b * static_cast<i128>(V2);  // checked below
    // exact comparison of lhs * 2^48 >= rhs_num without overflow:
    const i128 hi = rhs_num >> (2 * kThetaShift);
    const i128 lo = rhs_num & ((static_cast<i128>(1) << (2 * kThetaShift)) - 1);
    if (lhs != hi) return lhs > hi;
    return lo == 0;
}

int64_t largest_feasible(int64_t n, int64_t S, int64_t V2, int64_t eta, int64_t tq) {
    // Eq. 11 closed form (per-request moments, R3) as the starting point, then exact fix-up.
    const double th = static_cast<double>(tq) / static_cast<double>(1LL << kThetaShift);
    const double sv = std::sqrt(static_cast<double>(V2));
    const double x = (std::sqrt(th * th * static_cast<double>(V2) +
                                4.0 * static_cast<double>(S) * static_cast<double>(n) * static_cast<double>(eta)) -
                      th * sv) / (2.0 * static_cast<double>(S));
    int64_t b = static_cast<int64_t>(std::floor(x * x));
    if (b < 0) b = 0;
    while (b >= 1 && !feasible(b, n, S, V2, eta, tq)) --b;
    while (feasible(b + 1, n, S, V2, eta, tq)) ++b;
    return b;
}

struct WinRec {
    int64_t n, sl, sl2, so, so2;
};

}  // namespace

struct dbk_sched {
    dbk_sched_config cfg;
    int64_t tq = 0;
    int64_t t = 0, eta = 0, L0 = 0, bq = 0;
    int32_t b = 0, b_mem = 0, b_sla = 0, low = 0, high = 0;
    std::deque<WinRec> win;
    WinRec tot{0, 0, 0, 0, 0};
    std::deque<std::pair<int64_t, int64_t>> sla;  // (step_ns, n_active)
    int64_t sla_ns = 0, sla_b = 0;

    void push_window(const WinRec &r) {
        win.push_back(r);
        tot.n += r.n; tot.sl += r.sl; tot.sl2 += r.sl2; tot.so += r.so; tot.so2 += r.so2;
        while (win.size() > 1 && tot.n - win.front().n >= cfg.w_len) {
            const WinRec o = win.front();
            win.pop_front();
            tot.n -= o.n; tot.sl -= o.sl; tot.sl2 -= o.sl2; tot.so -= o.so; tot.so2 -= o.so2;
        }
    }
    void moments(int64_t &n, int64_t &S, int64_t &V2) const {
        n = tot.n;
        S = tot.sl + tot.so;
        V2 = (n * tot.sl2 - tot.sl * tot.sl) + (n * tot.so2 - tot.so * tot.so);
    }
};

extern "C" {

dbk_status dbk_theta_q(double eps_m, int64_t *out) {
    if (!out) return dbk::fail(DBK_EINVAL, "theta_q: null output");
    if (!(eps_m > 0.0 && eps_m <= 0.5)) return dbk::fail(DBK_EINVAL, "eps_M must be in (0, 0.5]");
    const double th = normal_quantile(1.0 - eps_m);  // theta = Theta^{-1}(1 - eps_M)
    *out = static_cast<int64_t>(std::floor(th * static_cast<double>(1LL << kThetaShift) + 0.5));
    if (*out < 0) *out = 0;
    return DBK_OK;
}

dbk_status dbk_b_quad(int64_t n, int64_t S, int64_t V2, int64_t eta, int64_t tq, int64_t *b_out) {
    if (!b_out || n < 1 || S < 1 || V2 < 0 || eta < 0 || tq < 0)
        return dbk::fail(DBK_EINVAL, "b_quad: bad arguments (empty window?)");
    *b_out = largest_feasible(n, S, V2, eta, tq);
    return DBK_OK;
}

dbk_status dbk_sched_create(const dbk_sched_config *cfg, dbk_sched **out) {
    if (!cfg || !out) return dbk::fail(DBK_EINVAL, "sched_create: null argument");
    const dbk_sched_config &c = *cfg;
    if (c.policy < 0 || c.policy > 3) return dbk::fail(DBK_EINVAL, "unknown policy %d", c.policy);
    if (c.policy == DBK_POLICY_STATIC) {
        if (c.b_static < 1) return dbk::fail(DBK_EINVAL, "b_static must be >= 1");
    } else if (c.b_min < 1 || c.b_min > c.b_max || c.b0 < 1 || c.b0 > c.b_max) {
        return dbk::fail(DBK_EINVAL, "need 1 <= B_min <= B_max and b0 in [1, B_max]");
    }
    if (c.policy == DBK_POLICY_MEMORY || c.policy == DBK_POLICY_COMBINED) {
        if (c.page_size < 1 || c.bytes_per_token < 1 || c.w_len < 1 || c.refresh_steps < 1)
            return dbk::fail(DBK_EINVAL, "memory policy needs page_size, bytes_per_token, w_len, refresh_steps >= 1");
        if (c.prior_n < 1 || c.prior_sum_lin + c.prior_sum_lout < 1)
            return dbk::fail(DBK_EINVAL, "memory policy needs a non-empty prior window");
    }
    if ((c.policy == DBK_POLICY_SLA || c.policy == DBK_POLICY_COMBINED) &&
        (c.alpha < 1 || c.delta < 1 || c.w_sla < 1 || c.eps_d_ms < 0))
        return dbk::fail(DBK_EINVAL, "SLA policy needs alpha, delta, w_sla >= 1 and eps_D >= 0");
    dbk_sched *s = new (std::nothrow) dbk_sched();
    if (!s) return dbk::fail(DBK_EINVAL, "out of host memory");
    s->cfg = c;
    if (c.policy == DBK_POLICY_MEMORY || c.policy == DBK_POLICY_COMBINED) {
        dbk_status st = dbk_theta_q(c.eps_m, &s->tq);
        if (st != DBK_OK) {
            delete s;
            return st;
        }
        s->push_window({c.prior_n, c.prior_sum_lin, c.prior_sum_lin_sq, c.prior_sum_lout, c.prior_sum_lout_sq});
    }
    s->b = s->b_mem = s->b_sla = (c.policy == DBK_POLICY_STATIC) ? c.b_static : c.b0;
    s->low = c.b_min;   // Alg. 2 line 1
    s->high = c.b_max;
    *out = s;
    return DBK_OK;
}

dbk_status dbk_sched_destroy(dbk_sched *s) {
    delete s;
    return DBK_OK;
}

dbk_status dbk_choose_batch_size(dbk_sched *s, const dbk_stats *g, int64_t mem_cap_bytes,
                                 double sla_ms, int32_t n_prefill, int32_t *b_out,
                                 int32_t *rationale_out) {
    if (!s || !g || !b_out) return dbk::fail(DBK_EINVAL, "choose_batch_size: null argument");
    if (g->n_active < 0 || g->n_finished < 0 || g->n_finished > g->n_active || n_prefill < 0)
        return dbk::fail(DBK_EINVAL, "choose_batch_size: inconsistent statistics");
    const dbk_sched_config &c = s->cfg;
    // every check before any state changes: a rejected call leaves the windows and bounds as
    // they were
    if ((c.policy == DBK_POLICY_MEMORY || c.policy == DBK_POLICY_COMBINED) && mem_cap_bytes < 0)
        return dbk::fail(DBK_EINVAL, "choose_batch_size: mem_cap_bytes < 0");
    if (!std::isfinite(sla_ms)) return dbk::fail(DBK_EINVAL, "choose_batch_size: sla_ms must be finite (<= 0: the configured D_SLA)");
    if (g->n_active > 0 && g->step_ns < 0) return dbk::fail(DBK_EINVAL, "choose_batch_size: step_ns < 0");
    if (g->n_finished > 0) {
        // lengths are >= 1, so sum >= count and sum of squares >= sum; and n * sum(l^2) >= sum(l)^2
        const i128 nf = g->n_finished;
        if (g->fin_sum_lin < g->n_finished || g->fin_sum_lout < g->n_finished || g->fin_sum_lin_sq < g->fin_sum_lin ||
            g->fin_sum_lout_sq < g->fin_sum_lout ||
            nf * g->fin_sum_lin_sq < static_cast<i128>(g->fin_sum_lin) * g->fin_sum_lin ||
            nf * g->fin_sum_lout_sq < static_cast<i128>(g->fin_sum_lout) * g->fin_sum_lout)
            return dbk::fail(DBK_EINVAL, "choose_batch_size: inconsistent finishing-request sums");
    }
    // telemetry windows
    if (g->n_finished > 0 && (c.policy == DBK_POLICY_MEMORY || c.policy == DBK_POLICY_COMBINED))
        s->push_window({g->n_finished, g->fin_sum_lin, g->fin_sum_lin_sq, g->fin_sum_lout, g->fin_sum_lout_sq});
    if (g->n_active > 0) {
        s->sla.emplace_back(g->step_ns, g->n_active);
        s->sla_ns += g->step_ns;
        s->sla_b += g->n_active;
        if (static_cast<int>(s->sla.size()) > c.w_sla) {
            s->sla_ns -= s->sla.front().first;
            s->sla_b -= s->sla.front().second;
            s->sla.pop_front();
        }
    }
    const int64_t n_decode = g->n_active - g->n_finished;  // N^d after retirement (R13)
    int32_t rationale = DBK_R_CARRY;
    if (c.policy == DBK_POLICY_STATIC) {
        s->t += 1;
        s->b = c.b_static;
        *b_out = s->b;
        if (rationale_out) *rationale_out = DBK_R_STATIC;
        return DBK_OK;
    }
    if (c.policy == DBK_POLICY_MEMORY || c.policy == DBK_POLICY_COMBINED) {
        const int64_t cap_pages = mem_cap_bytes / (static_cast<int64_t>(c.page_size) * c.bytes_per_token);
        s->eta = cap_pages * c.page_size;  // R4: eta in tokens
        int64_t n, S, V2;
        s->moments(n, S, V2);
        if (s->t % c.refresh_steps == 0) {  // R12: L0 "updated online periodically"
            s->bq = largest_feasible(n, S, V2, s->eta, s->tq);
            s->L0 = s->bq > 0 ? static_cast<int64_t>((static_cast<i128>(n) * s->eta - static_cast<i128>(s->bq) * S) / n)
                              : s->eta;  // R10
        }
        // Algorithm 1
        int64_t bm = s->b_mem;                                   // line 4
        if (n_decode > 0 && n_prefill > 0) {                     // line 5
            bm = static_cast<int64_t>((static_cast<i128>(s->eta - s->L0) * n) / S);  // line 6
            bm = std::min<int64_t>(std::max<int64_t>(bm, n_decode), c.b_max);      // line 7
            rationale = DBK_R_MEMORY;
        }
        s->b_mem = static_cast<int32_t>(bm);
    }
    if ((c.policy == DBK_POLICY_SLA || c.policy == DBK_POLICY_COMBINED) && !s->sla.empty()) {
        // Algorithm 2, integer ns (R14, R15)
        const double dms = sla_ms > 0 ? sla_ms : c.d_sla_ms;
        const int64_t d_ns = std::llround(dms * 1e6), e_ns = std::llround(c.eps_d_ms * 1e6);
        const int64_t cnt = static_cast<int64_t>(s->sla.size());
        const int64_t b_bar = (2 * s->sla_b + cnt) / (2 * cnt);  // line 4, round half up
        int64_t lo = s->low, hi = s->high, nlo, nhi;
        if (s->sla_ns > cnt * (d_ns + e_ns)) {           // line 5: tau_bar > D + eps_D
            nhi = std::max<int64_t>(b_bar, lo + c.alpha);  // line 6
            nlo = std::max<int64_t>(lo - c.delta, c.b_min); // line 7
        } else if (s->sla_ns < cnt * (d_ns - e_ns)) {    // line 8: tau_bar < D - eps_D
            nlo = std::min<int64_t>(b_bar, hi - c.alpha);  // line 9
            nhi = std::min<int64_t>(hi + c.delta, c.b_max); // line 10
        } else {
            nhi = std::min<int64_t>(b_bar + c.alpha / 2, c.b_max);  // line 12
            nlo = std::max<int64_t>(b_bar - c.alpha / 2, c.b_min);  // line 13
        }
        nlo = std::min<int64_t>(std::max<int64_t>(nlo, c.b_min), c.b_max);  // R14
        nhi = std::min<int64_t>(std::max<int64_t>(nhi, c.b_min), c.b_max);
        if (nlo > nhi) std::swap(nlo, nhi);
        int64_t bt = (nlo + nhi) / 2;                                              // line 15
        bt = std::min<int64_t>(std::max<int64_t>(bt, n_decode), c.b_max);          // line 16
        s->low = static_cast<int32_t>(nlo);
        s->high = static_cast<int32_t>(nhi);
        s->b_sla = static_cast<int32_t>(bt);
        if (c.policy == DBK_POLICY_SLA) rationale = DBK_R_SLA;
    }
    if (c.policy == DBK_POLICY_MEMORY) {
        s->b = s->b_mem;
    } else if (c.policy == DBK_POLICY_SLA) {
        s->b = s->b_sla;
    } else {  // b* = min{b_mem, b_SLA}
        s->b = std::min(s->b_mem, s->b_sla);
        rationale = s->b_mem < s->b_sla ? DBK_R_MEMORY : (s->b_sla < s->b_mem ? DBK_R_SLA : DBK_R_MIN);
    }
    s->t += 1;
    *b_out = s->b;
    if (rationale_out) *rationale_out = rationale;
    return DBK_OK;
}

dbk_status dbk_sched_get_state(dbk_sched *s, dbk_sched_state *o) {
    if (!s || !o) return dbk::fail(DBK_EINVAL, "sched_get_state: null argument");
    o->t = s->t;
    o->eta = s->eta;
    o->L0 = s->L0;
    o->b_quad = s->bq;
    o->theta_q = s->tq;
    s->moments(o->win_n, o->win_S, o->win_V2);
    o->b = s->b;
    o->b_mem = s->b_mem;
    o->b_sla = s->b_sla;
    o->b_low = s->low;
    o->b_high = s->high;
    o->sla_count = static_cast<int32_t>(s->sla.size());
    return DBK_OK;
}

}  // extern "C"
