#!/usr/bin/env python
"""Summarise an LX_TB2_TRACE dump: per pass, CTA start skew, arrival spread, barrier exit latency."""
import sys

import numpy as np

data = open(sys.argv[1], "rb").read()
off = 0
calls = []
while off < len(data):
    grid, npass = np.frombuffer(data, dtype=np.int32, count=2, offset=off)
    off += 8
    a = np.frombuffer(data, dtype=np.uint64, count=npass * grid * 3, offset=off).reshape(npass, grid, 3)
    off += a.nbytes
    calls.append(a)
a = calls[-1].astype(np.int64)
t0 = a[0, :, 0].min()
for p in range(a.shape[0]):
    st, ar, ex = a[p, :, 0], a[p, :, 1], a[p, :, 2]
    if (st == 0).all():
        break
    print("pass %2d start %8.1f..%8.1f  arrive min/med/p90/max %8.1f %8.1f %8.1f %8.1f  exit max %8.1f  "
          "(work med %6.1f us, tail %5.1f us, barrier %5.1f us)" % (
              p, (st.min() - t0) / 1e3, (st.max() - t0) / 1e3, (ar.min() - t0) / 1e3,
              (np.median(ar) - t0) / 1e3, (np.percentile(ar, 90) - t0) / 1e3, (ar.max() - t0) / 1e3,
              (ex.max() - t0) / 1e3, np.median(ar - st) / 1e3, (ar.max() - np.median(ar)) / 1e3,
              (ex.max() - ar.max()) / 1e3))
