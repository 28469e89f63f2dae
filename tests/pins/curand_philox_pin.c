/* Test pin (not product, not oracle): exposes cuRAND's own Philox4x32-10 block function
 * (curand_philox4x32_x.h, compiled for the host) so the oracle's Philox can be checked
 * on arbitrary counters and keys.  Built by tests/test_oracle_rng.py with g++. */
#include <vector_types.h>
#define QUALIFIERS static inline
#include <curand_philox4x32_x.h>
extern "C" void pin_philox(const unsigned *ctr, const unsigned *key, unsigned *out) {
    uint4 c = {ctr[0], ctr[1], ctr[2], ctr[3]};
    uint2 k = {key[0], key[1]};
    uint4 r = curand_Philox4x32_10(c, k);
    out[0] = r.x; out[1] = r.y; out[2] = r.z; out[3] = r.w;
}
