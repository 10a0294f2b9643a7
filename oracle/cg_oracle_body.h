/*
 * cg_oracle_body.h -- precision-generic body of the CPU oracle.
 *
 * TEST INFRASTRUCTURE ONLY.  Included twice by cg_oracle.c with
 *   REAL = double, SFX(x) = x##_f64     and     REAL = float, SFX(x) = x##_f32.
 * Every function restates one piece of the reference path (cellgrid 0.1.0,
 * paths relative to /root/reference/pkg/src/cellgrid/) in plain C with the
 * same operation order, so that -ffp-contract=off reproduces the numba
 * (fastmath off) results bit for bit.
 */

/* spatial.py:99-116 (build_grid geometry) + pool.py:102-110 (max_diameter,
 * bounding_box).  Extremes are taken in the pool dtype and widened to f64,
 * exactly as numpy's col.min()/max() followed by np.array(..., float64). */
int SFX(cgo_geometry)(int64_t n, const REAL *px, const REAL *py, const REAL *pz,
                      const REAL *diam, double interaction_radius, int64_t box_cap,
                      double *box_length, double origin[3], int64_t dims[3],
                      int64_t *num_boxes)
{
    if (n <= 0) return CGO_ERR_EMPTY;
    REAL dmax = diam[0];
    REAL lo[3] = {px[0], py[0], pz[0]}, hi[3] = {px[0], py[0], pz[0]};
    for (int64_t i = 1; i < n; ++i) {
        if (diam[i] > dmax) dmax = diam[i];
        const REAL p[3] = {px[i], py[i], pz[i]};
        for (int a = 0; a < 3; ++a) {
            if (p[a] < lo[a]) lo[a] = p[a];
            if (p[a] > hi[a]) hi[a] = p[a];
        }
    }
    double L = (double)dmax;
    if (!isnan(interaction_radius)) {          /* NaN encodes "None" */
        if (!(interaction_radius > 0)) return CGO_ERR_RADIUS;
        if (interaction_radius > L) L = interaction_radius;   /* max(ir, L) */
    }
    int64_t nb = 1;
    for (int a = 0; a < 3; ++a) {
        const double l = (double)lo[a], h = (double)hi[a];
        origin[a] = l - L;
        dims[a] = (int64_t)floor((h - l) / L) + 3;
        nb *= dims[a];
    }
    *box_length = L;
    *num_boxes = nb;
    return nb > box_cap ? CGO_ERR_GRID_OVERFLOW : CGO_OK;
}

/* kernels.py:107-129 box_ids_parallel (== spatial.py:130-136 numpy builder). */
void SFX(cgo_box_ids)(int64_t n, const REAL *px, const REAL *py, const REAL *pz,
                      double box_length, const double origin[3], const int64_t dims[3],
                      int64_t *out)
{
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        const double p[3] = {(double)px[i], (double)py[i], (double)pz[i]};
        int64_t c[3];
        for (int a = 0; a < 3; ++a) {
            int64_t k = (int64_t)floor((p[a] - origin[a]) / box_length);
            if (k < 0) k = 0;
            else if (k >= dims[a]) k = dims[a] - 1;
            c[a] = k;
        }
        out[i] = (c[0] * dims[1] + c[1]) * dims[2] + c[2];
    }
}

/* kernels.py:196-258 _sum_forces_sorted + :261-277 _write_displacement for
 * one agent whose stencil candidates are cand[0:m].  keep[] is scratch of the
 * same capacity.  Returns nk (colliding pairs) and adds degenerate pairs. */
static int64_t SFX(agent_force)(int64_t i, const int64_t *cand, int64_t m, int64_t *keep,
                                const REAL *px, const REAL *py, const REAL *pz,
                                const REAL *radii, const REAL *adherence,
                                const uint64_t *uid, const REAL *par,
                                REAL *out_dx, REAL *out_dy, REAL *out_dz,
                                int64_t *ndeg_out)
{
    const REAL zero = par[CGO_PAR_ZERO], kappa = par[CGO_PAR_KAPPA],
               gamma = par[CGO_PAR_GAMMA];
    const REAL xi = px[i], yi = py[i], zi = pz[i], ri = radii[i];
    int64_t nk = 0;
    for (int64_t t = 0; t < m; ++t) {             /* pass 1, kernels.py:196-205 */
        const int64_t j = cand[t];
        const REAL dx = xi - px[j], dy = yi - py[j], dz = zi - pz[j];
        const REAL dist = SQRT(dx * dx + dy * dy + dz * dz);
        const REAL delta = (ri + radii[j]) - dist;
        if (delta > zero) keep[nk++] = j;
    }
    /* uid-ascending order (kernels.py:206-225; uids unique => any sort) */
    for (int64_t a = 1; a < nk; ++a) {
        const int64_t v = keep[a];
        const uint64_t kv = uid[v];
        int64_t b = a - 1;
        while (b >= 0 && uid[keep[b]] > kv) { keep[b + 1] = keep[b]; --b; }
        keep[b + 1] = v;
    }
    REAL fx = zero, fy = zero, fz = zero;
    int64_t ndeg = 0;
    for (int64_t t = 0; t < nk; ++t) {            /* pass 2, kernels.py:230-257 */
        const int64_t j = keep[t];
        const REAL dx = xi - px[j], dy = yi - py[j], dz = zi - pz[j];
        const REAL dist = SQRT(dx * dx + dy * dy + dz * dz);
        const REAL rj = radii[j];
        const REAL rsum = ri + rj;
        const REAL delta = rsum - dist;
        const REAL req = (ri * rj) / rsum;
        const REAL mag = kappa * delta - gamma * SQRT(req * delta);
        if (dist > zero) {
            const REAL s = mag / dist;
            fx = fx + s * dx;
            fy = fy + s * dy;
            fz = fz + s * dz;
        } else {
            ++ndeg;
            const uint64_t ui = uid[i], uj = uid[j];
            double u[3];
            cgo_degenerate_dir(ui < uj ? ui : uj, ui < uj ? uj : ui, u);
            const double sign = ui < uj ? 1.0 : -1.0;
            /* tmp[0] = mag * (sign * u): f64 product rounded into the pool dtype */
            REAL tmp;
            tmp = (REAL)((double)mag * (sign * u[0])); fx = fx + tmp;
            tmp = (REAL)((double)mag * (sign * u[1])); fy = fy + tmp;
            tmp = (REAL)((double)mag * (sign * u[2])); fz = fz + tmp;
        }
    }
    /* _write_displacement, kernels.py:261-277 */
    const REAL norm = SQRT(fx * fx + fy * fy + fz * fz);
    if (norm <= par[CGO_PAR_ADH_SCALE] * adherence[i]) {
        out_dx[i] = zero; out_dy[i] = zero; out_dz[i] = zero;
    } else {
        REAL s = par[CGO_PAR_TIMESTEP];
        if (norm * s > par[CGO_PAR_MAX_DISP]) s = par[CGO_PAR_MAX_DISP] / norm;
        out_dx[i] = fx * s; out_dy[i] = fy * s; out_dz[i] = fz * s;
    }
    *ndeg_out += ndeg;
    return nk;
}

/* kernels.py:280-333 force_phase_serial / force_phase_parallel, with the
 * linked-cell stencil walk of kernels.py:148-173 replaced by an equivalent
 * CSR walk (box_start/box_members list each box's agents; chain order is
 * unobservable after the uid sort).  Optional per-agent m / nk outputs. */
void SFX(cgo_force_phase)(int64_t n, const REAL *px, const REAL *py, const REAL *pz,
                          const REAL *radii, const REAL *adherence, const uint64_t *uid,
                          const int64_t *box_index, const int64_t dims[3],
                          const int64_t *box_start, const int64_t *box_members,
                          int64_t cand_cap, const double params[7], int threads,
                          REAL *out_dx, REAL *out_dy, REAL *out_dz,
                          int32_t *m_out, int32_t *nk_out, int64_t counters[3])
{
    REAL par[7];
    for (int k = 0; k < 7; ++k) par[k] = (REAL)params[k];
    const int64_t dimx = dims[0], dimy = dims[1], dimz = dims[2];
    int64_t evals = 0, cands = 0, ndeg = 0;
    if (cand_cap < 1) cand_cap = 1;
    #pragma omp parallel num_threads(threads > 0 ? threads : 1) reduction(+ : evals, cands, ndeg)
    {
        int64_t *cand = (int64_t *)malloc(sizeof(int64_t) * (size_t)cand_cap);
        int64_t *keep = (int64_t *)malloc(sizeof(int64_t) * (size_t)cand_cap);
        #pragma omp for schedule(dynamic, 256)
        for (int64_t i = 0; i < n; ++i) {
            const int64_t flat = box_index[i];
            const int64_t iz = flat % dimz, rest = flat / dimz;
            const int64_t iy = rest % dimy, ix = rest / dimy;
            const int64_t x0 = ix > 0 ? ix - 1 : 0, x1 = ix + 1 < dimx ? ix + 1 : dimx - 1;
            const int64_t y0 = iy > 0 ? iy - 1 : 0, y1 = iy + 1 < dimy ? iy + 1 : dimy - 1;
            const int64_t z0 = iz > 0 ? iz - 1 : 0, z1 = iz + 1 < dimz ? iz + 1 : dimz - 1;
            int64_t m = 0;
            for (int64_t ax = x0; ax <= x1; ++ax)
                for (int64_t ay = y0; ay <= y1; ++ay) {
                    const int64_t base = (ax * dimy + ay) * dimz;
                    for (int64_t az = z0; az <= z1; ++az) {
                        const int64_t b = base + az;
                        for (int64_t t = box_start[b]; t < box_start[b + 1]; ++t) {
                            const int64_t j = box_members[t];
                            if (j != i) cand[m++] = j;
                        }
                    }
                }
            int64_t nd = 0;
            const int64_t nk = SFX(agent_force)(i, cand, m, keep, px, py, pz, radii, adherence,
                                                uid, par, out_dx, out_dy, out_dz, &nd);
            if (m_out) m_out[i] = (int32_t)m;
            if (nk_out) nk_out[i] = (int32_t)nk;
            cands += m;
            evals += nk;
            ndeg += nd;
        }
        free(cand);
        free(keep);
    }
    counters[0] = evals;
    counters[1] = cands;
    counters[2] = ndeg;
}

/* Brute-force all-pairs displacement oracle (mechanics.py:186-233): O(n^2),
 * uid-ordered summation.  Used to pin the grid path on tiny pools. */
void SFX(cgo_all_pairs)(int64_t n, const REAL *px, const REAL *py, const REAL *pz,
                        const REAL *radii, const REAL *adherence, const uint64_t *uid,
                        const double params[7], REAL *out_dx, REAL *out_dy, REAL *out_dz,
                        int64_t counters[3])
{
    REAL par[7];
    for (int k = 0; k < 7; ++k) par[k] = (REAL)params[k];
    int64_t *cand = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 1 ? n : 1));
    int64_t *keep = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 1 ? n : 1));
    int64_t evals = 0, ndeg = 0;
    for (int64_t i = 0; i < n; ++i) {
        int64_t m = 0;
        for (int64_t j = 0; j < n; ++j) if (j != i) cand[m++] = j;
        evals += SFX(agent_force)(i, cand, m, keep, px, py, pz, radii, adherence, uid, par,
                                  out_dx, out_dy, out_dz, &ndeg);
    }
    free(cand);
    free(keep);
    counters[0] = evals;
    counters[1] = n * (n - 1);
    counters[2] = ndeg;
}
