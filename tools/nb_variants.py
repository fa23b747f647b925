"""A/B of the bulk-staged odd-width network kernel (netbulk.cu) against the
cp.async tile kernel (net_sort.cuh) on the cfg2 odd-n cells.

    python tools/nb_variants.py [reps] [force...]     # on the GPU

Each round runs bench.py with the default dispatch, with NSG_NET_TILE_ONLY=1
(every shape on the tile kernel) and with NSG_NB_FORCE=<c> for each listed
configuration c (1 = A, 2 = B, 3 = C in netbulk.cu: every odd n on that
configuration), and prints GB/s per cell.  The per-shape choice in
netbulk.cu (nb_choice) comes from these runs (profiles/round2/netbulk.md).
"""

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def run(env_extra):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "bench.py", "--ns", "5,7,9,11,13,15", "--workloads", "none", "--no-e2e",
                        "--no-cpu", "--steps", "5"], cwd=ROOT, env=env, capture_output=True, text=True)
    line = [l for l in r.stdout.splitlines() if l.startswith("{")]
    if not line:
        raise SystemExit(r.stderr[-2000:])
    return json.loads(line[-1])["per_kernel_gbs"]


if __name__ == "__main__":
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    forces = sys.argv[2:]
    for i in range(reps):
        out = {"round": i, "default": run({}), "tile_only": run({"NSG_NET_TILE_ONLY": "1"})}
        for f in forces:
            out[f"force{f}"] = run({"NSG_NB_FORCE": f})
        print(json.dumps(out), flush=True)
