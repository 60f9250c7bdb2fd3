"""Build A/B variants of libstamg_b200.so into abl/<name>.so (compile-time knobs
via STAMG_NVCC_EXTRA); select one at run time with STAMG_LIB=abl/<name>.so.
Usage: python tools/ab_build.py name='-DKNOB=1 ...' [name2=...]"""
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    os.makedirs(os.path.join(ROOT, "abl"), exist_ok=True)
    for arg in sys.argv[1:]:
        name, flags = arg.split("=", 1)
        os.environ["STAMG_NVCC_EXTRA"] = flags
        import importlib

        from paper_2010_04559_b200 import build as B
        importlib.reload(B)
        B.build(force=True)
        shutil.copy(B.OUT, os.path.join(ROOT, "abl", name + ".so"))
        print(name, flags)
    os.environ["STAMG_NVCC_EXTRA"] = ""
    from paper_2010_04559_b200 import build as B
    importlib.reload(B)
    B.build(force=True)


if __name__ == "__main__":
    main()
