"""Generate tests/golden/refine_golden.txt from the REFERENCE library (test infrastructure).

Run here, where /root/reference exists, after `make -C oracle`:

    python tests/golden/make_refine_golden.py

Compiles tests/golden/gen_refine.cpp against the reference headers and the reference
library compiled in place (oracle/_ref/liblongctx_ref.so), runs it, and writes its
output (calibration inputs, configs, and the reference's refine_plan / offline_search
results and CriticalSet / SparsityPlan JSON) to refine_golden.txt.  It also copies the
reference's own committed JSON outputs proj/out/sparsity/critical_set.json and
proj/out/refine/plan_refined.json, proj/out/sparsity/prefill_selections.json (files
the reference CLI wrote) as ref_*.json: their
text pins the JSON formatting (the nlohmann bundled here prints arrays inline, the
reference's build one element per line).  The GPU box only reads the committed files.
"""
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/proj"
NLOHMANN = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty"


def main():
    lib = os.path.join(ROOT, "oracle", "_ref")
    if not os.path.exists(os.path.join(lib, "liblongctx_ref.so")):
        sys.exit("build the reference first: make -C oracle")
    exe = os.path.join("/tmp", "gen_refine")
    subprocess.run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-I", REF + "/core/include",
                    "-I", NLOHMANN, os.path.join(HERE, "gen_refine.cpp"), "-L", lib,
                    "-llongctx_ref", f"-Wl,-rpath,{lib}", "-o", exe], check=True)
    out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout
    with open(os.path.join(HERE, "refine_golden.txt"), "w") as f:
        f.write(out)
    dc = subprocess.run([exe, "dcpp"], check=True, capture_output=True, text=True).stdout
    with open(os.path.join(HERE, "dcpp_golden.txt"), "w") as f:
        f.write(dc)
    shutil.copy(REF + "/out/sparsity/critical_set.json", os.path.join(HERE, "ref_critical_set.json"))
    shutil.copy(REF + "/out/refine/plan_refined.json", os.path.join(HERE, "ref_plan_refined.json"))
    shutil.copy(REF + "/out/sparsity/prefill_selections.json",
                os.path.join(HERE, "ref_prefill_selections.json"))
    print("wrote refine_golden.txt,", len(out), "bytes")


if __name__ == "__main__":
    main()
