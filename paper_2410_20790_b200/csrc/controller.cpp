// controller.cpp -- Online Truncation Threshold Adjustment (§3.4,
// P:171-181): BST and IBST, host side, one observation
// per site per step (reading R15).  Update rule, constants and restart
// policy are readings R16: bisection on [lo, hi] from
// theta_max/2; s > T+eps lowers hi, s < T-eps raises lo; freeze in band or
// when hi-lo <= theta_res; IBST restarts the bracket every `cycle`
// observations keeping theta as the first probe.  All arithmetic in double;
// thresholds handed out as float (round-to-nearest).
#include <cmath>
#include <new>
#include <vector>

#include "sparsetem.h"

struct st_controller {
    st_ctl_config cfg;
    int n;
    std::vector<double> theta, lo, hi;
    std::vector<int32_t> frozen, count;
};

extern "C" st_status st_controller_create(const st_ctl_config *cfg, int32_t n_sites, st_controller **out) {
    if (!cfg || !out || n_sites < 1) return ST_ERR_ARG;
    if (cfg->policy < 0 || cfg->policy > 2) return ST_ERR_ARG;
    if (cfg->policy != 0 && (!(cfg->theta_max > 0.0f) || !(cfg->theta_res > 0.0f) || cfg->theta_res >= cfg->theta_max ||
                             cfg->eps <= 0.0f || cfg->T - cfg->eps < 0.0f || cfg->T + cfg->eps > 1.0f))
        return ST_ERR_ARG;
    if (cfg->policy == 2 && cfg->cycle < 1) return ST_ERR_ARG;
    st_controller *c = new (std::nothrow) st_controller();
    if (!c) return ST_ERR_OOM;
    c->cfg = *cfg;
    c->n = n_sites;
    const double t0 = cfg->policy == 0 ? (double)cfg->theta_fixed : (double)cfg->theta_max / 2.0;
    c->theta.assign(n_sites, t0);
    c->lo.assign(n_sites, 0.0);
    c->hi.assign(n_sites, (double)cfg->theta_max);
    c->frozen.assign(n_sites, 0);
    c->count.assign(n_sites, 0);
    *out = c;
    return ST_OK;
}

extern "C" st_status st_controller_observe(st_controller *c, const int64_t *site_active, const int64_t *site_pixels) {
    if (!c || !site_active || !site_pixels) return ST_ERR_ARG;
    const double T = c->cfg.T, eps = c->cfg.eps, res = c->cfg.theta_res, tmax = c->cfg.theta_max;
    for (int i = 0; i < c->n; i++) {
        if (site_pixels[i] <= 0) continue;
        if (site_active[i] < 0 || site_active[i] > site_pixels[i]) return ST_ERR_ARG;
        if (c->cfg.policy == 0) continue;
        const double s = 1.0 - (double)site_active[i] / (double)site_pixels[i];
        if (!c->frozen[i]) {
            if (s > T + eps) c->hi[i] = c->theta[i];
            else if (s < T - eps) c->lo[i] = c->theta[i];
            const bool band = s >= T - eps && s <= T + eps;
            if (band || c->hi[i] - c->lo[i] <= res) c->frozen[i] = 1;
            else c->theta[i] = (c->lo[i] + c->hi[i]) / 2.0;
        }
        if (c->cfg.policy == 2 && ++c->count[i] >= c->cfg.cycle) {
            c->count[i] = 0;
            c->lo[i] = 0.0;
            c->hi[i] = tmax;
            c->frozen[i] = 0;
        }
    }
    return ST_OK;
}

extern "C" st_status st_controller_thresholds(const st_controller *c, float *out) {
    if (!c || !out) return ST_ERR_ARG;
    for (int i = 0; i < c->n; i++) out[i] = (float)c->theta[i];
    return ST_OK;
}

extern "C" st_status st_controller_state(const st_controller *c, double *theta, double *lo, double *hi,
                                         int32_t *frozen) {
    if (!c) return ST_ERR_ARG;
    for (int i = 0; i < c->n; i++) {
        if (theta) theta[i] = c->theta[i];
        if (lo) lo[i] = c->lo[i];
        if (hi) hi[i] = c->hi[i];
        if (frozen) frozen[i] = c->frozen[i];
    }
    return ST_OK;
}

extern "C" void st_controller_destroy(st_controller *c) { delete c; }
