// Independent pin for oracle/philox.py: cuRAND's own Philox4x32-10
// (CUDA toolkit header curand_philox4x32_x.h, whose mulhilo32 has a host branch),
// compiled for the HOST with g++.  Reads "c0 c1 c2 c3 k0 k1" (hex) per line on
// stdin, prints the four output words (hex) per line.
#include <cstdio>
#include <vector_types.h>
#define QUALIFIERS static inline
#include <curand_philox4x32_x.h>

int main() {
  unsigned c0, c1, c2, c3, k0, k1;
  while (std::scanf("%x %x %x %x %x %x", &c0, &c1, &c2, &c3, &k0, &k1) == 6) {
    uint4 c; c.x = c0; c.y = c1; c.z = c2; c.w = c3;
    uint2 k; k.x = k0; k.y = k1;
    uint4 o = curand_Philox4x32_10(c, k);
    std::printf("%08x %08x %08x %08x\n", o.x, o.y, o.z, o.w);
  }
  return 0;
}
