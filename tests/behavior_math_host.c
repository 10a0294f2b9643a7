// Host build of paper_2105_00039_b200/csrc/behavior_math.h for the CPU tests
// (tests/test_behavior_math.py): gcc -O2 -ffp-contract=off -shared.
#include "../paper_2105_00039_b200/csrc/behavior_math.h"

using namespace cgb;

extern "C" {
void bm_cbrt64(long n, const double *x, double *y) { for (long i = 0; i < n; ++i) y[i] = cbrt_svml(x[i]); }
void bm_cbrt32(long n, const float *x, float *y) { for (long i = 0; i < n; ++i) y[i] = cbrtf_svml(x[i]); }
void bm_log1p(long n, const double *x, double *y) { for (long i = 0; i < n; ++i) y[i] = log1p_glibc(x[i]); }
void bm_philox_raw(uint64_t k0, uint64_t k1, long n, uint64_t *out)
{
    Philox g;
    philox_init(g, k0, k1);
    for (long i = 0; i < n; ++i) out[i] = philox_next(g);
}
void bm_normals(uint64_t k0, uint64_t k1, long n, double *out)
{
    Philox g;
    philox_init(g, k0, k1);
    for (long i = 0; i < n; ++i) out[i] = standard_normal(g);
}
void bm_unit_vectors(long n, const uint64_t *uid, uint64_t step, double *out)
{
    for (long i = 0; i < n; ++i) unit_vector(uid[i], step, out + 3 * i);
}
}
