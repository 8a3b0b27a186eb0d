"""Kernel split of one config-1 dense FCS call (100^3 fp64, J=1000, D=1) for ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2106_13062_b200 as st  # noqa: E402
from paper_2106_13062_b200 import configs  # noqa: E402

c = configs.C1
x = torch.from_numpy(configs.c1_tensor(c)).cuda()
fams = st.families_for(list(c.dims), st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed))
packed = st.packed_families(fams)
t = st.DenseTensor(list(c.dims), x.flatten())
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    st.fcs_dense_batched(t, fams, packed=packed)
torch.cuda.synchronize()
