"""Copy the reference test suite next to the alias conftest (run in the build container, where the
reference checkout exists; the copy is git-ignored and travels to the GPU box with gpurun).

    python tools/refsuite/fetch.py [/root/reference/pkg]
    gpurun -- 'cd tools/refsuite && python -m pytest tests -q -rA -p no:cacheprovider'
"""
import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
src = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg"
dst = os.path.join(HERE, "tests")
if os.path.exists(dst):
    shutil.rmtree(dst)
shutil.copytree(os.path.join(src, "tests"), dst)
if os.path.isdir(os.path.join(src, "configs")):
    shutil.copytree(os.path.join(src, "configs"), os.path.join(HERE, "configs"), dirs_exist_ok=True)
print("copied", sorted(os.listdir(dst)))
