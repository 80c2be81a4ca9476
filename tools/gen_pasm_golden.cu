// gen_pasm_golden.cu -- writes tests/golden/pasm_uniform.json: the PASM draw's
// uniform u_i = (x0 >> 8) * 2^-24 for fixed (seed, batch_seq, i), with x0 the first
// word of Philox4x32-10(counter = {i, seq lo, seq hi, 0}, key = {seed lo, seed hi})
// (R20, "probabilistically redistributed").  x0 is computed by
// NVIDIA cuRAND's curand_Philox4x32_10 compiled for the host -- an implementation
// independent of both oracle/ and libargus -- so the golden pins the oracle's counter
// layout and word choice, not just its Philox rounds (which the Random123 KATs pin).
//   nvcc -o /tmp/gen_pasm_golden tools/gen_pasm_golden.cu && /tmp/gen_pasm_golden > tests/golden/pasm_uniform.json
#include <cstdint>
#include <cstdio>
#define QUALIFIERS static inline __host__ __device__
#include <curand_philox4x32_x.h>

int main() {
  struct T { unsigned long long seed, seq; unsigned i; };
  const T cases[] = {{0ull, 0ull, 0u},          {0ull, 0ull, 1u},           {0ull, 1ull, 0u},
                     {1ull, 0ull, 0u},          {2511ull, 0ull, 7u},         {2511ull, 3ull, 7u},
                     {7ull, 3ull, 5u},          {0x123456789abcdefull, 0x100000002ull, 4095u},
                     {11ull, 0ull, 69999u},     {0xffffffffffffffffull, 0xffffffffull, 0xffffffffu}};
  printf("{\n  \"citation\": \"DESIGN.md R20 (PASM sampling, P:299, P:351): u = (x0 >> 8) * 2^-24 with x0 = word 0 of "
         "Philox4x32-10(counter = {i, seq mod 2^32, seq >> 32, 0}, key = {seed mod 2^32, seed >> 32}); x0 computed by "
         "cuRAND curand_Philox4x32_10 (host build, tools/gen_pasm_golden.cu). u_m = x0 >> 8, u = u_m / 2^24.\",\n");
  printf("  \"cases\": [\n");
  const int n = sizeof(cases) / sizeof(cases[0]);
  for (int t = 0; t < n; ++t) {
    const T& c = cases[t];
    uint4 ctr = make_uint4(c.i, (unsigned)(c.seq & 0xffffffffu), (unsigned)(c.seq >> 32), 0u);
    uint2 key = make_uint2((unsigned)(c.seed & 0xffffffffu), (unsigned)(c.seed >> 32));
    uint4 x = curand_Philox4x32_10(ctr, key);
    printf("    {\"seed\": %llu, \"seq\": %llu, \"i\": %u, \"x0\": \"%08x\", \"x1\": \"%08x\", \"u_m\": %u}%s\n", c.seed,
           c.seq, c.i, x.x, x.y, x.x >> 8, t + 1 < n ? "," : "");
  }
  printf("  ]\n}\n");
  return 0;
}
