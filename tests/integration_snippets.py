"""The ctypes binding documented in INTEGRATION.md §2, extracted so tests run
exactly what a maintainer would paste (the snippet cannot drift from the
header unnoticed)."""
import os
import re

from conftest import REPO


def snippets():
    txt = open(os.path.join(REPO, "INTEGRATION.md")).read()
    sec = txt[txt.index("## 2. C-ABI"):]
    return re.findall(r"```python\n(.*?)```", sec, flags=re.S)


def load_binding(extra_ns=None):
    """Execute the §2 blocks in order from the repo root; returns the
    namespace (L = the CDLL with the documented argtypes, als_half_step)."""
    ns = dict(extra_ns or {})
    cwd = os.getcwd()
    os.chdir(REPO)
    try:
        for block in snippets():
            exec(compile(block, "INTEGRATION.md", "exec"), ns)
    finally:
        os.chdir(cwd)
    return ns
