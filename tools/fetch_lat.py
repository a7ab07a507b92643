"""Publication -> fetch latency of BLOCK's cross-cluster values (mailbox
written by the producer -> copied into the consumer's shared slot by the
fetcher warp), from a block_trace2 dump with the publication trace."""
import sys
import numpy as np
d = np.load(sys.argv[1])
ftr = d["ftr"].astype(np.float64)
ptr = d["ptr"].astype(np.float64)
items = d["items"]
ok = (ftr > 0) & (ptr[items[:, 0]] > 0)
lat = ftr[ok] - ptr[items[ok, 0]]
print(f"items {len(ftr)} with both stamps {ok.sum()}")
print("publish -> fetched latency ns: p5 %.0f p25 %.0f p50 %.0f p75 %.0f p95 %.0f max %.0f" %
      tuple(np.percentile(lat, [5, 25, 50, 75, 95, 100])))
