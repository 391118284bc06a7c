"""Source-level check of the programmatic-dependent-launch contract (launch.cuh):
a kernel launched with the PDL attribute may start before the previous kernel on
its stream has finished, so it must execute griddepcontrol.wait (pdl_entry())
before it reads anything that kernel produced.  Every kernel passed to
pdl_launch -- and the CTA-pair GEMM launched with the attribute directly -- must
call pdl_entry() in its body."""
import glob
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2104_04473_b200", "csrc")


def sources():
    return {p: open(p).read() for p in glob.glob(os.path.join(CSRC, "*.cu"))}


def _skip_parens(src, i):
    depth = 0
    while True:
        if src[i] == "(":
            depth += 1
        elif src[i] == ")":
            depth -= 1
            if depth == 0:
                return i + 1
        i += 1


def kernel_bodies(src):
    """name -> body text of every __global__ function."""
    out = {}
    for m in re.finditer(r"__global__", src):
        i = m.end()
        name = None
        while name is None:
            t = re.match(r"\s*(\w+)", src[i:])
            word, i = t.group(1), i + t.end()
            if word in ("__launch_bounds__", "__maxnreg__"):
                i = _skip_parens(src, src.index("(", i))
            elif word != "void":
                name = word
        i = src.index("{", i)
        depth, j = 0, i
        while True:
            if src[j] == "{":
                depth += 1
            elif src[j] == "}":
                depth -= 1
                if depth == 0:
                    break
            j += 1
        out.setdefault(name, "")
        out[name] += src[i:j + 1]
    return out


def test_every_pdl_launched_kernel_waits():
    srcs = sources()
    bodies = {}
    for s in srcs.values():
        bodies.update(kernel_bodies(s))
    launched = set()
    for s in srcs.values():
        for m in re.finditer(r"pdl_launch\(\s*([A-Za-z_]\w*)", s):
            launched.add(m.group(1))
    # the CTA-pair GEMM sets cudaLaunchAttributeProgrammaticStreamSerialization itself
    launched.add("tc_gemm_kernel")
    # pdl_launch(kern, ...) with a local variable: resolve to the kernel templates it is bound to
    launched -= {"kern", "k"}
    launched |= {"ln_fwd_kernel"}
    missing = [k for k in sorted(launched) if k in bodies and "pdl_entry()" not in bodies[k]]
    unknown = [k for k in sorted(launched) if k not in bodies]
    assert not unknown, unknown
    assert not missing, missing
    assert len(launched) >= 20


def test_pdl_entry_waits_for_the_previous_grid():
    src = open(os.path.join(CSRC, "launch.cuh")).read()
    body = src[src.index("void pdl_entry()"):]
    body = body[:body.index("}")]
    assert "griddepcontrol.wait" in body and "griddepcontrol.launch_dependents" in body
