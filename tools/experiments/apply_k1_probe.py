"""Temporarily instrument fcs_dense_fx_kernel with probe modes (not for merge):
ST_FX_PROBE=1 replaces the shared-memory atomic by a register op (loads +
arithmetic only), =2 replaces the global loads by synthesised values
(atomics + arithmetic only). Restore with `git checkout` of fcs_dense.cu."""
p = 'paper_2106_13062_b200/csrc/fcs_dense.cu'
s = open(p).read()
s = s.replace('template <int NV, int SPLIT, int THREADS, bool kFull>\n__global__',
              'template <int NV, int SPLIT, int THREADS, bool kFull, int MODE = 0>\n__global__')
s = s.replace('      if (vbase + lane + 32 * j < nvec) dst[j] = __ldcs(src + vbase + lane + 32 * j);',
              '''      if (vbase + lane + 32 * j < nvec) {
        if (MODE == 2) {
          const float z = static_cast<float>((lane + j) ^ static_cast<uint32_t>(fib & 7));
          dst[j] = make_float4(z, -z, 0.5f * z, 0.25f);
        } else {
          dst[j] = __ldcs(src + vbase + lane + 32 * j);
        }
      }''')
old_atom = '''          asm volatile("atom.shared.add.s32 %0, [%1], %2;"
                       : "=r"(old)
                       : "r"(base_c + (e << 2)), "r"(q));'''
assert old_atom in s
s = s.replace(old_atom, '''          if (MODE == 1) {
            old = static_cast<int32_t>(base_c + (e << 2)) ^ q;
          } else {
            asm volatile("atom.shared.add.s32 %0, [%1], %2;"
                         : "=r"(old)
                         : "r"(base_c + (e << 2)), "r"(q));
          }''')
s = s.replace('  ovf = (ovf_acc >> 31) | ((rng_acc >> 23) != 0);',
              '  ovf = (ovf_acc >> 31) | ((rng_acc >> 23) != 0);\n  if (MODE != 0) ovf = (ovf_acc == 0x12345u) && (rng_acc == 0x54321u);')
s = s.replace('    default: return fcs_dense_fx_kernel<8, 1, 512, true>;',
              '''    case 11: return fcs_dense_fx_kernel<8, 1, 512, true, 1>;
    case 12: return fcs_dense_fx_kernel<8, 1, 512, true, 2>;
    default: return fcs_dense_fx_kernel<8, 1, 512, true>;''')
s = s.replace('  p->nv = sizeof(Tin) == 4 ? fx_nv(a) : 0;',
              '''  p->nv = sizeof(Tin) == 4 ? fx_nv(a) : 0;
  if (p->nv == 8 && std::getenv("ST_FX_PROBE")) p->nv = 10 + std::atoi(std::getenv("ST_FX_PROBE"));''')
s = s.replace('#include <algorithm>\n', '#include <algorithm>\n#include <cstdlib>\n', 1)
open(p, 'w').write(s)
