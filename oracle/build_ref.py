"""ORACLE - test infrastructure only.

Compile the UNMODIFIED reference package (``/root/reference/pkg/src/kifmm3d``,
all modules except the CLI) with Cython + gcc into ``oracle/_ref/kifmm3d/``
(a namespace package of extension modules; git-ignored, but it travels to
the GPU box with the snapshot).  No reference source is copied: Cython reads
the files where they lie and only the compiled ``.so`` files land in
``oracle/_ref``.  ``_hot.pyx`` is built with the reference's own flags
(``-O3 -fopenmp``, pkg/setup.py:16-25).

Run: ``python oracle/build_ref.py`` (skips silently when /root/reference is
absent, e.g. on the GPU box, where the prebuilt files are used).
"""

import glob
import os
import sys

SRC = "/root/reference/pkg/src/kifmm3d"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_ref")
SKIP = {"__main__", "__init__", "cli"}


def main():
    if not os.path.isdir(SRC):
        print("build_ref: reference tree absent; using prebuilt oracle/_ref if any")
        return 0
    from Cython.Build import cythonize
    from setuptools import Extension, setup
    os.environ.setdefault("CC", "/usr/bin/gcc")
    os.environ.setdefault("LDSHARED", "/usr/bin/gcc -shared")
    exts = []
    for f in sorted(glob.glob(SRC + "/*.py")) + [SRC + "/_hot.pyx"]:
        name = os.path.splitext(os.path.basename(f))[0]
        if name in SKIP:
            continue
        hot = name == "_hot"
        exts.append(Extension("kifmm3d." + name, [f],
                              extra_compile_args=["-O3", "-fopenmp"] if hot else ["-O2"],
                              extra_link_args=["-fopenmp"] if hot else []))
    import shutil
    import tempfile
    build_tmp = tempfile.mkdtemp(prefix="kifmm_ref_build_")   # generated C stays out of the repo
    setup(name="kifmm3d_ref_compiled",
          ext_modules=cythonize(exts, build_dir=os.path.join(build_tmp, "c"), language_level=3,
                                quiet=True),
          script_args=["build_ext", "--build-lib", OUT, "--build-temp",
                       os.path.join(build_tmp, "o")])
    shutil.rmtree(build_tmp, ignore_errors=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
