"""Every profile / evidence file the docs cite exists in the tree (DESIGN.md,
README.md, ROUND_SUMMARY.md, profiles/README.md, tools/experiments/README.md):
a backticked name containing r01_/r02_ is expanded ({a,b} and * globs) and
must match at least one file under profiles/ (or the path as written)."""
import glob
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DOCS = ["DESIGN.md", "README.md", "ROUND_SUMMARY.md", "profiles/README.md", "tools/experiments/README.md"]


def expand(tok):
    m = re.search(r"\{([^{}]*)\}", tok)
    if not m:
        return [tok]
    out = []
    for alt in m.group(1).split(","):
        out += expand(tok[:m.start()] + alt + tok[m.end():])
    return out


def references(doc):
    with open(os.path.join(ROOT, doc)) as f:
        text = f.read()
    for tok in re.findall(r"`([^`]+)`", text):
        for word in tok.split():
            word = word.strip(",;:()")
            if re.search(r"\br0[12]_", word) and "." in word.split("/")[-1] or re.search(r"r0[12]_.*\*", word):
                yield word


@pytest.mark.parametrize("doc", DOCS)
def test_cited_profiles_exist(doc):
    missing = []
    for ref in references(doc):
        for name in expand(ref):
            cands = [os.path.join(ROOT, name), os.path.join(ROOT, "profiles", os.path.basename(name))]
            if not any(glob.glob(c) for c in cands):
                missing.append(name)
    assert not missing, missing


@pytest.mark.parametrize("doc", DOCS)
def test_cited_source_paths_exist(doc):
    with open(os.path.join(ROOT, doc)) as f:
        text = f.read()
    missing = []
    for tok in re.findall(r"`([^`]+)`", text):
        for word in tok.split():
            word = word.strip(",;:()")
            if re.match(r"(tools|tests|include|oracle|seeded_inputs|paper_2508_13397_b200)/[\w./{},*-]+$", word):
                for name in expand(word.split(":")[0]):
                    if not glob.glob(os.path.join(ROOT, name)):
                        missing.append(name)
    assert not missing, missing
