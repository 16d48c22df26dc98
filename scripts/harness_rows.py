"""Harness closure rows: configs/sweep_consolidation.toml's cells plus
the cluster_baseline.toml partition on B200s, served by the reference-semantics loop
with the decode step priced by the B200-measured step table; writes ROW_FIELDS rows
(harness.py:33-45) and prints shared vs partitioned TPOT p50.

  python scripts/harness_rows.py --out tests/golden/b200_consolidation_rows.csv
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_02599_b200 import harness, pricing
from paper_2603_02599_b200.sun_types import GpuSpec

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# configs/cluster_shared.toml [cost] (prefill half; the decode step comes from the B200 table)
COST = pricing.CostParams(prefill_flops_per_token=16060000000.0, prefill_fixed_overhead=0.029316666666666696,
                          decode_fixed_overhead=0.005429770674636779, dequant_compute_penalty=1.2422027153707458,
                          mfu=0.7530766952319238, mbu=0.9527915328513344)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", default=os.path.join(ROOT, "tests", "golden", "b200_steps_8b_bf16.json"))
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    hdr, pts = pricing.load_step_points(args.grid)
    backend = pricing.MeasuredBackend(pts, hdr["kv_bytes_per_token"])
    gpu = GpuSpec.b200(6463.3, 1666.0)
    rows = []
    t0 = time.time()
    for cell in harness.consolidation_cells(gpu):
        rows.append(harness.run_cell(cell, COST, backend, "b200-measured:" + os.path.basename(args.grid)))
    with open(args.out, "w") as fh:
        harness.write_rows(rows, fh)
    print(f"{len(rows)} rows in {time.time() - t0:.1f} s -> {args.out}")
    for r in rows:
        print(f"  {r['decode_pool_mode']:8s} D={r['decode_pool_size']} alpha={r['alpha']} osl={r['osl']}: "
              f"tpot_p50 {float(r['tpot_p50_s']) * 1e3 if r['tpot_p50_s'] != '' else float('nan'):7.2f} ms, "
              f"tok/s/decode-GPU {float(r['throughput_per_decode_gpu_tok_s'] or 'nan'):8.0f} {r['error']}")


if __name__ == "__main__":
    main()
