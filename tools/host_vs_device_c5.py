"""C5 through the host-buffer C-ABI path (row-chunked upload; the sketch AND
the first power product A^T Y summed under the upload) against the
device-resident path (the reference's operation order, which matched the
unmodified reference at full size: profiles/r02_parity_full.jsonl), on the
same A with the same Philox Omega.  Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1502_05366_b200 as R
from paper_1502_05366_b200.testmat import gen_test_matrix_device

m, n, k, p, q = 200000, 20000, 500, 10, 2
eng = R.Engine(0)
A, st = gen_test_matrix_device(eng, m, n, np.exp(-np.arange(3685) / 100.0), seed=5)
Ud = torch.empty(m * k, dtype=torch.float64, device="cuda")
Vd = torch.empty(n * k, dtype=torch.float64, device="cuda")
Sd = torch.empty(k, dtype=torch.float64, device="cuda")
eng.device_rsvd(R.RSVD_V2, A.data_ptr(), m, n, m, k, p, q, 1, R.Omega.philox(777), Ud.data_ptr(), Sd.data_ptr(),
                Vd.data_ptr())
eng.synchronize()
ed = eng.device_rel_error(A.data_ptr(), m, n, Ud.data_ptr(), Sd.data_ptr(), Vd.data_ptr(), k)
Ah = torch.empty(m * n, dtype=torch.float64, pin_memory=True)
Ah.copy_(A)
Uh = torch.empty(m * k, dtype=torch.float64, pin_memory=True)
Vh = torch.empty(n * k, dtype=torch.float64, pin_memory=True)
Sh = torch.empty(k, dtype=torch.float64, pin_memory=True)
eng.host_rsvd_ptr(R.RSVD_V2, Ah.data_ptr(), m, n, m, k, p, q, 1, R.Omega.philox(777), Uh.data_ptr(), Sh.data_ptr(),
                  Vh.data_ptr())
U2, V2, S2 = Uh.cuda(), Vh.cuda(), Sh.cuda()
eh = eng.device_rel_error(A.data_ptr(), m, n, U2.data_ptr(), S2.data_ptr(), V2.data_ptr(), k)
sd, sh = Sd.cpu().numpy(), Sh.numpy()
print(json.dumps(dict(config="C5 host path vs device path", sigma_max_rel_diff=float(np.max(np.abs(sh - sd) / sd)),
                      rel_fro_error_host=eh, rel_fro_error_device=ed, residual_ratio=eh / ed)), flush=True)
