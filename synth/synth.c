/*
 * Seeded synthetic key generators shared by the tests, the bench and smoke().
 * Holds NONE of the method's arithmetic: it only produces input arrays, once,
 * on the host; the CUDA path and the oracle both receive the same bytes.
 * Recipe: a counter-based stream r(seed, stream, i), unit
 * uniforms U = (r >> 11) * 2^-53 in [0,1), Box-Muller normals,
 * inverse-CDF exponentials.  libm exp/log/cos are not bit-portable
 * across machines, which does not matter: both sides consume these bytes.
 */
#include <stdint.h>
#include <math.h>

static uint64_t sm_fin(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static uint64_t stream_base(uint64_t seed, uint64_t stream)
{
    return sm_fin(seed ^ ((stream + 1) * 0xD1B54A32D192ED03ULL));
}

static uint64_t r_at(uint64_t base, uint64_t i) { return sm_fin(base + (i + 1) * 0x9E3779B97F4A7C15ULL); }
static double u_at(uint64_t base, uint64_t i) { return (double)(r_at(base, i) >> 11) * 0x1.0p-53; }

static double normal_at(uint64_t b0, uint64_t b1, uint64_t i)
{
    double u1 = u_at(b0, i), u2 = u_at(b1, i);
    return sqrt(-2.0 * log(1.0 - u1)) * cos(6.283185307179586 * u2);
}

/* dist: 0 uniform[0,1), 1 normal(0,1), 2 exponential(1), 3 lognormal(0,1),
 *       4 mixture of 8 gaussians + 10% one repeated value, 5 exp(700 U^4),
 *       6 uint64 uniform over [0, 2^64).  out holds n 8-byte keys. */
void synth_generate(int dist, uint64_t seed, uint64_t n, void *outp)
{
    uint64_t b0 = stream_base(seed, 0), b1 = stream_base(seed, 1);
    uint64_t b2 = stream_base(seed, 2), b3 = stream_base(seed, 3);
    double mu[8], sg[8];
    uint64_t bm = stream_base(seed, 10), bs = stream_base(seed, 11);
    for (int c = 0; c < 8; c++) {
        mu[c] = -1000.0 + 2000.0 * u_at(bm, (uint64_t)c);
        sg[c] = 1.0 + 49.0 * u_at(bs, (uint64_t)c);
    }
    double *xd = (double *)outp;
    uint64_t *xu = (uint64_t *)outp;
    int64_t nn = (int64_t)n;
#pragma omp parallel for schedule(static)
    for (int64_t ii = 0; ii < nn; ii++) {
        uint64_t i = (uint64_t)ii;
        switch (dist) {
        case 0: xd[i] = u_at(b0, i); break;
        case 1: xd[i] = normal_at(b0, b1, i); break;
        case 2: xd[i] = -log(1.0 - u_at(b0, i)); break;
        case 3: xd[i] = exp(normal_at(b0, b1, i)); break;
        case 4: {
            int c = (int)(u_at(b2, i) * 8.0);
            double x = mu[c] + sg[c] * normal_at(b0, b1, i);
            if (u_at(b3, i) < 0.1) x = mu[0];
            xd[i] = x;
            break;
        }
        case 5: { double u = u_at(b0, i); double u2 = u * u; xd[i] = exp(700.0 * (u2 * u2)); break; }
        default: xu[i] = r_at(b0, i); break;
        }
    }
}
