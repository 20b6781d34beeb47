"""Build alternative libb200rt variants (same ABI, other -D flags) for A/B runs."""
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, ".")
from paper_2303_11103_b200 import _native as N  # noqa: E402


def build(name, defines):
    cmd = N.nvcc_command(out=N.LIB_PATH.replace("libb200rt.so", f"libb200rt_{name}.so"))
    for d in defines:
        cmd.insert(1, f"-D{d}")
    r = subprocess.run(cmd, capture_output=True, text=True)
    return name, r.returncode, r.stderr[-300:]


if __name__ == "__main__":
    specs = {}
    for arg in sys.argv[1:]:
        name, _, defs = arg.partition("=")
        specs[name] = [d for d in defs.split(",") if d]
    with ThreadPoolExecutor(len(specs)) as ex:
        for name, rc, err in ex.map(lambda kv: build(*kv), specs.items()):
            print(name, rc, err)
