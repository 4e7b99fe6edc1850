"""Build an A/B variant of libsfk.so with extra nvcc defines for some sources:

    python tools/build_variant.py NAME "-DFOO=1 -DBAR=2" csrc_file.cu [more.cu]

Writes paper_1711_02473_b200/libsfk_NAME.so from the current objects with the
listed sources recompiled (use with SFK_LIBRARY / tools/ab_cfg_libs.sh).
"""
import os
import shlex
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1711_02473_b200 import _build as B  # noqa: E402


def main():
    name, defines, files = sys.argv[1], shlex.split(sys.argv[2]), sys.argv[3:]
    B.build_native()
    vdir = os.path.join(B.BUILD, "variant_" + name)
    os.makedirs(vdir, exist_ok=True)
    objs = []
    for o in sorted(os.listdir(B.BUILD)):
        if o.endswith(".o"):
            objs.append(os.path.join(B.BUILD, o))
    for f in files:
        src = os.path.join(B.CSRC, os.path.basename(f))
        obj = os.path.join(vdir, os.path.splitext(os.path.basename(f))[0] + ".o")
        subprocess.run([B.nvcc()] + B.NVCC_FLAGS + defines + ["-c", src, "-o", obj], check=True)
        objs = [obj if os.path.basename(x) == os.path.basename(obj) else x for x in objs]
    out = os.path.join(B.PKG, "libsfk_%s.so" % name)
    subprocess.run([B.nvcc()] + B.ARCH + ["-shared", "-o", out] + objs
                   + ["-cudart", "static", "-ldl"], check=True)
    print(out)


if __name__ == "__main__":
    main()
