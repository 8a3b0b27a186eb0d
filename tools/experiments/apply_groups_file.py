"""Probe (not for merge): ST_FX_GROUPS_FILE=<D x NV x 4 uint8> replaces the
fx_group_kernel search with groups read from a file. Restore with git checkout."""
p = 'paper_2106_13062_b200/csrc/fcs_dense.cu'
s = open(p).read()
old = '''      fx_group_kernel<<<a.D, 32 * 4 * nv_full, 0, st>>>(packed, a.fam_stride, a.i0_shift, nv_full,
                                                       groups);
      FCS_CUDA_TRY(cudaGetLastError());'''
assert old in s
s = s.replace(old, '''      if (const char* gf = std::getenv("ST_FX_GROUPS_FILE")) {
        static std::vector<uint8_t> hg;
        if (hg.empty()) {
          FILE* fp = std::fopen(gf, "rb");
          hg.resize(static_cast<size_t>(a.D) * nv_full * 4);
          if (!fp || std::fread(hg.data(), 1, hg.size(), fp) != hg.size()) return ST_EINVAL;
          std::fclose(fp);
        }
        FCS_CUDA_TRY(cudaMemcpyAsync(groups, hg.data(), hg.size(), cudaMemcpyHostToDevice, st));
      } else {
        fx_group_kernel<<<a.D, 32 * 4 * nv_full, 0, st>>>(packed, a.fam_stride, a.i0_shift, nv_full,
                                                         groups);
        FCS_CUDA_TRY(cudaGetLastError());
      }''', 1)
s = s.replace('#include <algorithm>\n', '#include <algorithm>\n#include <cstdio>\n#include <vector>\n', 1)
open(p, 'w').write(s)
