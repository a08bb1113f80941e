"""C5 tensor-core phase cycles (library built with -DQX_TC_TIMING, via
QX_NATIVE_LIB): one template search per mode (tc_f2 = argv[1])."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2509_19974_b200 as P
from paper_2509_19974_b200 import _native as N, workloads as W

tpl, st, off, sn2 = W.c5()
td, sd = torch.from_numpy(tpl).cuda(), torch.from_numpy(st).cuda()
with N.option("tc_f2", int(sys.argv[1]) if len(sys.argv) > 1 else 0):
    P.batch.template_search_summary(td, sd, P.sign(), P.sign())
    torch.cuda.synchronize()
