/*
 * oracle/oracle.c — plain, slow, obviously-correct float64 CPU oracle for the
 * FinRL-Podracer (arXiv 2111.05188) vectorised-rollout hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product path (paper_2111_05188_b200/) never links, imports or executes it,
 * and shares no code, header, table or constant generator with it.
 *
 * Citations: "P:Lx" = /root/reference/PAPER.md line x, "S:Lx" = SPEC.md line x,
 * "R#k" = reading k of DESIGN.md §3 (the readings table, copied from
 * SURVEY.md §8(c)).
 *
 * Compiled with -O2 -ffp-contract=off (no FMA contraction, IEEE binary64 on
 * x86-64 SSE2), so every expression below is evaluated exactly as written,
 * left to right.
 *
 * Pins: every function is pinned by tests/test_oracle_pins.py against values
 * the paper/spec fix (files under tests/golden), closed forms, invariants or brute
 * force.  There is no "parity unpinned" function in this file.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------- */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11 "Parallel random numbers:
 * as easy as 1, 2, 3", Random123).  R#14: the action noise stream.  Written
 * out from the published round function: two 32x32->64 multiplies per round,
 * Weyl key schedule.  Pinned by the Random123 known-answer vectors.          */
static void mulhilo32(uint32_t a, uint32_t b, uint32_t* hi, uint32_t* lo) {
    uint64_t p = (uint64_t)a * (uint64_t)b;
    *hi = (uint32_t)(p >> 32);
    *lo = (uint32_t)p;
}

void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        uint32_t hi0, lo0, hi1, lo1;
        mulhilo32(M0, c0, &hi0, &lo0);
        mulhilo32(M1, c2, &hi1, &lo1);
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += W0; k1 += W1;          /* key bump after each round (unused after the last) */
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Standard normals for one (env, step): R#14.
 * counter = (env_global, step_lo, quad, step_hi), key = (seed_lo, seed_hi).
 * Box–Muller (Box & Muller 1958): u1 = (x0+1)·2^-32 ∈ (0,1], u2 = x1·2^-32,
 * z0 = sqrt(-2 ln u1) cos(2π u2), z1 = sqrt(-2 ln u1) sin(2π u2); the second
 * pair from (x2, x3).  Ticker i takes quad i/4, component i%4.               */
void orc_normals(uint64_t seed, int64_t env_global, uint64_t step, int n, double* z) {
    const double two_m32 = 1.0 / 4294967296.0;
    const double two_pi = 6.283185307179586476925286766559;
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    for (int quad = 0; quad * 4 < n; ++quad) {
        uint32_t ctr[4] = {(uint32_t)env_global, (uint32_t)step, (uint32_t)quad,
                           (uint32_t)(step >> 32)};
        uint32_t x[4];
        orc_philox4x32_10(ctr, key, x);
        double zz[4];
        for (int pair = 0; pair < 2; ++pair) {
            double u1 = ((double)x[2 * pair] + 1.0) * two_m32;
            double u2 = (double)x[2 * pair + 1] * two_m32;
            double rad = sqrt(-2.0 * log(u1));
            zz[2 * pair] = rad * cos(two_pi * u2);
            zz[2 * pair + 1] = rad * sin(two_pi * u2);
        }
        for (int c = 0; c < 4 && quad * 4 + c < n; ++c) z[quad * 4 + c] = zz[c];
    }
}

/* ------------------------------------------------------------------------- */
/* Action map, R#6 ("k <= h_max"):
 * a = sgn(u) * floor(|u| * h_max + 1/2)  (round half away from zero).       */
int orc_map_action(double u, int h_max) {
    double m = floor(fabs(u) * (double)h_max + 0.5);
    int a = (int)m;
    return u < 0.0 ? -a : a;
}

/* ------------------------------------------------------------------------- */
/* Configuration shared by the env functions.                                */
typedef struct {
    int n_envs, n_stocks, n_feat, horizon, h_max;
    int n_agents;           /* envs split into n_agents contiguous equal groups */
    double C0, cost, scale, gamma;
    uint64_t seed;
    int64_t env_offset;     /* global id of env 0 (Philox counter, R#14) */
    int64_t T_data;
} orc_cfg;

/* Per-env carried state: balance b, shares h,
 * episode start row s, step-in-episode k (t = s + k), account value v,
 * discounted-return accumulators for the fitness J (Eq. 1, R#15).   */
typedef struct {
    double* cash;      /* [N]   b_t                                   */
    double* asset;     /* [N]   v_t = b_t + p_t^T h_t                 */
    double* disc;      /* [N]   sum_k gamma^k r_k of running episode  */
    double* gpow;      /* [N]   gamma^k                               */
    double* ep_ret;    /* [N]   disc of last completed episode        */
    int32_t* hold;     /* [N][n] h_t (env-major)                      */
    int64_t* start;    /* [N]   s                                     */
    int64_t* k;        /* [N]   k                                     */
} orc_state;

/* reset, S:L155–163 / R#17: b = C0, h = 0, t = s. */
static void env_reset(const orc_cfg* c, orc_state* st, int e) {
    st->cash[e] = c->C0;
    st->asset[e] = c->C0;
    st->disc[e] = 0.0;
    st->gpow[e] = 1.0;
    st->k[e] = 0;
    for (int i = 0; i < c->n_stocks; ++i) st->hold[(int64_t)e * c->n_stocks + i] = 0;
}

void orc_reset(const orc_cfg* c, orc_state* st) {
    for (int e = 0; e < c->n_envs; ++e) env_reset(c, st, e);
}

/* Observation, P:L220–226 (balance, shares, closing price, indicators) in
 * the S:L164–172 layout (R#9):
 *   o = [ b/C0, (h_i p_{t,i}/C0)_i, (p_{t,i}/p0_i)_i, (feat[t][c][i])_{c,i} ]
 * p0 = close at the episode start row s.  Length 1 + 2n + n f.             */
void orc_obs(const orc_cfg* c, const float* close, const float* feat,
             const orc_state* st, int e, double* o) {
    const int n = c->n_stocks, f = c->n_feat;
    const int64_t s = st->start[e], t = s + st->k[e];
    o[0] = st->cash[e] / c->C0;
    for (int i = 0; i < n; ++i) {
        double p = (double)close[t * n + i];
        o[1 + i] = (double)st->hold[(int64_t)e * n + i] * p / c->C0;
    }
    for (int i = 0; i < n; ++i)
        o[1 + n + i] = (double)close[t * n + i] / (double)close[s * n + i];
    for (int ch = 0; ch < f; ++ch)
        for (int i = 0; i < n; ++i)
            o[1 + 2 * n + ch * n + i] = (double)feat[(t * f + ch) * n + i];
}

/* One environment transition with integer actions a[n], Eqs. 3–4
 * and reward P:L230–234 Eq. 2, under readings R#1–5, R#8, R#10, R#18:
 *   sells (i ascending): q = min(h_i, -a_i); h_i -= q; b += (p_i q)(1-c)
 *   buys  (i ascending): unit = p_i (1+c); q = floor(b/unit), minus one if
 *         q*unit > b; q = max(0, min(a_i, q)); h_i += q; b -= q*unit
 *   v' = b + (sum_i p_{t+1,i} h_i);  r = scale (v' - v)
 *   fitness accumulators (Eq. 1): disc += gamma^k r; gamma^k *= gamma
 *   k += 1; done = (k == H) or (t+1 == T_data - 1); on done: record the
 *   terminal transition, ep_ret = disc, auto-reset.
 * Returns done; *reward gets r; *near_tie counts buy decisions whose
 * quotient b/unit lies within 1e-9 (relative) of an integer (R#19);
 * hold_post / cash_post (optional) get h_{t+1}, b_{t+1} before any reset.  */
int orc_env_step(const orc_cfg* c, const float* close, orc_state* st, int e,
                 const int32_t* a, double* reward, int64_t* near_tie,
                 int32_t* hold_post, double* cash_post, double* asset_post) {
    const int n = c->n_stocks;
    const int64_t t = st->start[e] + st->k[e];
    int32_t* h = st->hold + (int64_t)e * n;
    double cash = st->cash[e];
    const double one_minus_c = 1.0 - c->cost;
    const double one_plus_c = 1.0 + c->cost;
    /* selling set S (Eq. 3 "+ (p^S)^T k^S", Eq. 4 "- k^S", h >= 0) */
    for (int i = 0; i < n; ++i) {
        if (a[i] < 0) {
            int32_t q = -a[i] < h[i] ? -a[i] : h[i];
            double p = (double)close[t * n + i];
            h[i] -= q;
            cash = cash + (p * (double)q) * one_minus_c;
        }
    }
    /* buying set B (Eq. 3 "- (p^B)^T k^B", Eq. 4 "+ k^B"), b >= 0 (R#4) */
    for (int i = 0; i < n; ++i) {
        if (a[i] > 0) {
            double p = (double)close[t * n + i];
            double unit = p * one_plus_c;
            double x = cash / unit;
            double qmax = floor(x);
            if (qmax * unit > cash) qmax = qmax - 1.0;
            double r = floor(x + 0.5);
            if (near_tie && x >= 0.5 && fabs(x - r) <= 1e-9 * x) (*near_tie)++;
            double q = (double)a[i] < qmax ? (double)a[i] : qmax;
            if (q < 0.0) q = 0.0;
            h[i] += (int32_t)q;
            cash = cash - q * unit;
        }
    }
    /* account value at s_{t+1} (Eq. 2 first term) */
    double ph = 0.0;
    for (int i = 0; i < n; ++i) ph = ph + (double)close[(t + 1) * n + i] * (double)h[i];
    double v1 = cash + ph;
    double r = c->scale * (v1 - st->asset[e]);
    st->cash[e] = cash;
    st->asset[e] = v1;
    st->disc[e] = st->disc[e] + st->gpow[e] * r;
    st->gpow[e] = st->gpow[e] * c->gamma;
    st->k[e] += 1;
    int done = (st->k[e] == c->horizon) || (t + 1 == c->T_data - 1);
    *reward = r;
    if (hold_post) memcpy(hold_post, h, sizeof(int32_t) * (size_t)n);
    if (cash_post) *cash_post = cash;
    if (asset_post) *asset_post = v1;
    if (done) {
        st->ep_ret[e] = st->disc[e];
        env_reset(c, st, e);
    }
    return done;
}

/* ------------------------------------------------------------------------- */
/* Actor mean mu = W_L act(... act(W_1 o + b_1) ...) + b_L ("a function
 * that maps a state to an action vector"; R#12, R#13).  Weights in the
 * oracle's own unpadded row-major layout, float64:
 *   W_1 [H][obs_dim], b_1 [H], (W_l [H][H], b_l [H]) x (n_hidden-1),
 *   W_out [n][H], b_out [n], log_std [n].
 * act: 0 = ReLU, 1 = tanh.                                                   */
int64_t orc_actor_weight_count(int obs_dim, int n_hidden, int hidden, int n) {
    int64_t c = (int64_t)hidden * obs_dim + hidden;
    c += (int64_t)(n_hidden - 1) * ((int64_t)hidden * hidden + hidden);
    c += (int64_t)n * hidden + n + n;
    return c;
}

void orc_actor_mu(const double* w, int obs_dim, int n_hidden, int hidden, int n, int act,
                  const double* o, double* mu, double* scratch /* [2*hidden] */) {
    double* x = scratch;
    double* y = scratch + hidden;
    const double* p = w;
    int in_dim = obs_dim;
    const double* in = o;
    for (int l = 0; l < n_hidden; ++l) {
        const double* W = p;
        const double* b = p + (int64_t)hidden * in_dim;
        for (int j = 0; j < hidden; ++j) {
            double s = 0.0;
            for (int i = 0; i < in_dim; ++i) s = s + W[(int64_t)j * in_dim + i] * in[i];
            s = s + b[j];
            y[j] = act == 0 ? (s > 0.0 ? s : 0.0) : tanh(s);
        }
        p = b + hidden;
        in_dim = hidden;
        double* tmp = x; x = y; y = tmp;
        in = x;
    }
    const double* W = p;
    const double* b = p + (int64_t)n * hidden;
    for (int j = 0; j < n; ++j) {
        double s = 0.0;
        for (int i = 0; i < hidden; ++i) s = s + W[(int64_t)j * hidden + i] * in[i];
        mu[j] = s + b[j];
    }
}

/* Critic ("shared trunk -> actor head + critic head", R#22):
 * V = w_v . h_L + b_v, where h_L is the last hidden layer that orc_actor_mu
 * leaves in scratch (x after n_hidden swaps), summed in the head's order.
 * critic = [w_v (hidden), b_v].                                              */
double orc_critic_value(const double* critic, int n_hidden, int hidden, const double* scratch) {
    const double* h = scratch + ((n_hidden % 2) ? hidden : 0);
    double s = 0.0;
    for (int i = 0; i < hidden; ++i) s = s + critic[i] * h[i];
    return s + critic[hidden];
}

/* Gaussian policy head (R#12): raw = mu + exp(log_std) z,
 * log pi(raw) = sum_i (-z_i^2/2 - log_std_i - ln(2 pi)/2), u = tanh(raw).
 * deterministic: z = 0.                                                      */
double orc_sample(int n, const double* mu, const double* log_std, const double* z,
                  int deterministic, double* raw, double* u) {
    const double half_ln_2pi = 0.91893853320467274178032973640562;
    double lp = 0.0;
    for (int i = 0; i < n; ++i) {
        double zi = deterministic ? 0.0 : z[i];
        raw[i] = mu[i] + exp(log_std[i]) * zi;
        u[i] = tanh(raw[i]);
        lp = lp + (-0.5 * zi * zi - log_std[i] - half_ln_2pi);
    }
    return lp;
}

/* ------------------------------------------------------------------------- */
/* T-step rollout over all envs ("a batched environment ... takes a
 * batch of actions and returns a batch of transitions").  Envs are
 * independent, so the env loop may run on several threads; each env
 * is stepped sequentially in t.
 * mode: 0 = injected u [T][N][n] (float), 1 = replay a_int [T][N][n],
 *       2 = sample from the actor, 3 = deterministic actor (z = 0).
 * weights: [n_agents][orc_actor_weight_count] (modes 2, 3).
 * Outputs (any may be NULL):
 *   obs [T+1][N][obs_dim], mu/raw [T][N][n], logp/rew [T][N], done [T][N],
 *   a_out/hold_out [T][N][n], cash_out [T][N] (h_{t+1}, b_{t+1} of the
 *   transition, before any auto-reset).  Returns the number of near-tie
 *   buy decisions.                                                          */
int64_t orc_rollout(const orc_cfg* c, const float* close, const float* feat, orc_state* st,
                    int T, int mode, const float* u_inj, const int16_t* a_rep,
                    const double* weights, int n_hidden, int hidden, int act, uint64_t step0,
                    double* obs, double* mu_out, double* raw_out, double* logp_out,
                    double* rew_out, uint8_t* done_out, int32_t* a_out, int32_t* hold_out,
                    double* cash_out, const double* critic, double* val_out, double* asset_out, int nthreads) {
    const int N = c->n_envs, n = c->n_stocks, f = c->n_feat;
    const int od = 1 + 2 * n + n * f;
    const int64_t wcount = orc_actor_weight_count(od, n_hidden, hidden, n);
    const int per_agent = N / (c->n_agents > 0 ? c->n_agents : 1);
    int64_t ties = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : ties)
#endif
    for (int e = 0; e < N; ++e) {
        double* o = (double*)malloc(sizeof(double) * (size_t)od);
        double* mu = (double*)malloc(sizeof(double) * (size_t)n * 4);
        double* raw = mu + n;
        double* u = mu + 2 * n;
        double* z = mu + 3 * n;
        double* scratch = (double*)malloc(sizeof(double) * (size_t)(2 * (hidden > 0 ? hidden : 1)));
        int32_t* a = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
        const double* w = weights ? weights + (int64_t)(e / per_agent) * wcount : NULL;
        orc_obs(c, close, feat, st, e, o);
        if (obs) memcpy(obs + (int64_t)e * od, o, sizeof(double) * (size_t)od);
        for (int t = 0; t < T; ++t) {
            const int64_t te = (int64_t)t * N + e;
            double lp = 0.0;
            if (mode == 0) {
                for (int i = 0; i < n; ++i) a[i] = orc_map_action((double)u_inj[te * n + i], c->h_max);
            } else if (mode == 1) {
                for (int i = 0; i < n; ++i) a[i] = (int32_t)a_rep[te * n + i];
            } else {
                orc_actor_mu(w, od, n_hidden, hidden, n, act, o, mu, scratch);
                if (critic && val_out)
                    val_out[te] = orc_critic_value(critic + (int64_t)(e / per_agent) * (hidden + 1), n_hidden,
                                                   hidden, scratch);
                orc_normals(c->seed, c->env_offset + e, step0 + (uint64_t)t, n, z);
                const double* log_std = w + wcount - n;
                lp = orc_sample(n, mu, log_std, z, mode == 3, raw, u);
                for (int i = 0; i < n; ++i) a[i] = orc_map_action(u[i], c->h_max);
                if (mu_out) memcpy(mu_out + te * n, mu, sizeof(double) * (size_t)n);
                if (raw_out) memcpy(raw_out + te * n, raw, sizeof(double) * (size_t)n);
                if (logp_out) logp_out[te] = lp;
            }
            if (a_out) memcpy(a_out + te * n, a, sizeof(int32_t) * (size_t)n);
            double r;
            int64_t nt = 0;
            int d = orc_env_step(c, close, st, e, a, &r, &nt,
                                 hold_out ? hold_out + te * n : NULL,
                                 cash_out ? cash_out + te : NULL,
                                 asset_out ? asset_out + te : NULL);
            ties += nt;
            if (rew_out) rew_out[te] = r;
            if (done_out) done_out[te] = (uint8_t)d;
            orc_obs(c, close, feat, st, e, o);
            if (obs) memcpy(obs + ((int64_t)(t + 1) * N + e) * od, o, sizeof(double) * (size_t)od);
        }
        if (mode >= 2 && critic && val_out) {   /* bootstrap V(s_T) */
            orc_actor_mu(w, od, n_hidden, hidden, n, act, o, mu, scratch);
            val_out[(int64_t)T * N + e] =
                orc_critic_value(critic + (int64_t)(e / per_agent) * (hidden + 1), n_hidden, hidden, scratch);
        }
        free(o); free(mu); free(scratch); free(a);
    }
    return ties;
}

/* ------------------------------------------------------------------------- */
/* GAE (not in the paper; PPO P:L472 needs it, R#11):
 *   delta_t = r_t + gamma (1-d_t) V_{t+1} - V_t,   V_T = boot
 *   A_t     = delta_t + gamma lambda (1-d_t) A_{t+1},  A_T = 0
 *   R_t     = A_t + V_t
 * Also the magnitude recurrence used for tolerances:
 *   M_t = (|r_t| + gamma (1-d_t)|V_{t+1}| + |V_t|) + gamma lambda (1-d_t) M_{t+1}.
 * Layout [T][N], one column per env.                                        */
void orc_gae(int T, int N, const double* r, const double* v, const uint8_t* d,
             const double* boot, double gamma, double lam, double* adv, double* ret,
             double* mag) {
    for (int e = 0; e < N; ++e) {
        double a_next = 0.0, m_next = 0.0, v_next = boot[e];
        for (int t = T - 1; t >= 0; --t) {
            const int64_t i = (int64_t)t * N + e;
            double nd = d[i] ? 0.0 : 1.0;
            double delta = r[i] + gamma * nd * v_next - v[i];
            double a = delta + gamma * lam * nd * a_next;
            adv[i] = a;
            ret[i] = a + v[i];
            if (mag) {
                double m = (fabs(r[i]) + gamma * nd * fabs(v_next) + fabs(v[i])) + gamma * lam * nd * m_next;
                mag[i] = m;
                m_next = m;
            }
            a_next = a;
            v_next = v[i];
        }
    }
}

/* ------------------------------------------------------------------------- */
/* Fitness J (Eq. 1 "expected return (the fitness score)", R#15):
 * the mean over an agent's envs of the discounted return of the last
 * completed episode, summed in env order.                                   */
void orc_fitness(int N, int n_agents, const double* ep_ret, double* J) {
    int per = N / n_agents;
    for (int a = 0; a < n_agents; ++a) {
        double s = 0.0;
        for (int e = a * per; e < (a + 1) * per; ++e) s = s + ep_ret[e];
        J[a] = s / (double)per;
    }
}

/* Selector ("redistributes the agents with the highest scores to form
 * a new population", R#16): rank by (J desc, id asc); the first
 * k are elites and keep their weights; the eliminated slots, in ascending id,
 * receive elites in rank order, round-robin.  plan[g] = source agent of slot
 * g.  Returns 0, or -1 on bad arguments / non-finite fitness.       */
int orc_select_elite(int P, const double* J, int k, int32_t* plan) {
    if (P < 1 || k < 1 || k > P) return -1;
    for (int g = 0; g < P; ++g)
        if (!isfinite(J[g])) return -1;
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)P);
    for (int g = 0; g < P; ++g) order[g] = g;
    /* insertion sort: plainly a stable sort on J descending, id ascending */
    for (int i = 1; i < P; ++i) {
        int32_t x = order[i];
        int j = i - 1;
        while (j >= 0 && (J[order[j]] < J[x] || (J[order[j]] == J[x] && order[j] > x))) {
            order[j + 1] = order[j];
            --j;
        }
        order[j + 1] = x;
    }
    char* elite = (char*)calloc((size_t)P, 1);
    for (int r = 0; r < k; ++r) elite[order[r]] = 1;
    int next = 0;
    for (int g = 0; g < P; ++g) {
        if (elite[g]) {
            plan[g] = g;
        } else {
            plan[g] = order[next % k];
            ++next;
        }
    }
    free(order);
    free(elite);
    return 0;
}
