"""Temporarily instrument the grouped fcs_dense_fx_kernel with probe modes
(not for merge; restore with `git checkout` of fcs_dense.cu):
ST_FX_PROBE=1 replaces the shared-memory atomic by a register op (loads +
arithmetic), =2 synthesises the tensor values instead of loading them
(atomics + arithmetic), =3 uses red.shared.add (no returned value, no wrap
guard)."""
p = 'paper_2106_13062_b200/csrc/fcs_dense.cu'
s = open(p).read()
s = s.replace('template <int NV, int SPLIT, int THREADS, bool kFull, bool kGroup = false>\n__global__',
              'template <int NV, int SPLIT, int THREADS, bool kFull, bool kGroup = false, int MODE = 0>\n__global__')
old = '      for (int j = 0; j < NV; ++j) dst[j] = ld_stream(src + ((vmap[j / 4] >> (8 * (j % 4))) & 0xffu));'
assert old in s
s = s.replace(old, '''      for (int j = 0; j < NV; ++j) {
        if (MODE == 2) {
          const float z = static_cast<float>((lane + j) ^ static_cast<uint32_t>(fib & 7));
          dst[j] = make_float4(z, -z, 0.5f * z, 0.25f);
        } else {
          dst[j] = ld_stream(src + ((vmap[j / 4] >> (8 * (j % 4))) & 0xffu));
        }
      }''')
old_atom = '''          asm volatile("atom.shared.add.s32 %0, [%1], %2;"
                       : "=r"(old)
                       : "r"(base_c + (e << 2)), "r"(q));'''
assert old_atom in s
s = s.replace(old_atom, '''          if (MODE == 1) {
            old = static_cast<int32_t>(base_c + (e << 2)) ^ q;
          } else if (MODE == 3) {
            asm volatile("red.shared.add.s32 [%0], %1;" :: "r"(base_c + (e << 2)), "r"(q));
            old = 0;
          } else {
            asm volatile("atom.shared.add.s32 %0, [%1], %2;"
                         : "=r"(old)
                         : "r"(base_c + (e << 2)), "r"(q));
          }''')
old = '  ovf = (ovf_acc >> 31) | ((rng_acc >> 23) != 0);'
assert old in s
s = s.replace(old, old + '\n  if (MODE == 1 || MODE == 2) ovf = (ovf_acc == 0x12345u) && (rng_acc == 0x54321u);')
old = '      case 8: return fcs_dense_fx_kernel<8, 1, 512, true, true>;'
assert old in s
s = s.replace(old, '''      case 8:
        if (const char* m = std::getenv("ST_FX_PROBE")) {
          switch (std::atoi(m)) {
            case 1: return fcs_dense_fx_kernel<8, 1, 512, true, true, 1>;
            case 2: return fcs_dense_fx_kernel<8, 1, 512, true, true, 2>;
            case 3: return fcs_dense_fx_kernel<8, 1, 512, true, true, 3>;
            default: break;
          }
        }
        return fcs_dense_fx_kernel<8, 1, 512, true, true>;''')
open(p, 'w').write(s)
