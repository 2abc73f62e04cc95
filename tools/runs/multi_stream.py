"""K independent streams on one GPU (bench.multi_stream_run).  Usage: multi_stream.py c2 1 2 4:30 6:20
(K or K:chain blocks per stream)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2007_10798_b200 as rocp  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
for a in sys.argv[2:] or ["1", "2", "4"]:
    K, _, sm = a.partition(":")
    K = int(K)
    r = bench.multi_stream_run(rocp, cfg, K, 10, 3, chain_sms=int(sm or 0))
    print(f"K={K} sms/stream={r['chain_sms_per_stream']} aggregate {r['value']:.0f} slices/s, "
          f"{r['ms_per_round']:.3f} ms per round (wall {r['wall_ms']:.2f} ms, events {r['event_ms_max']:.2f} ms)", flush=True)
