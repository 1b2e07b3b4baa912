"""INTEGRATION.md's reference-side binding is real code: extract the C++
snippet, compile it against the reference's headers (/root/reference, present
in the build container only) and link it with the compiled reference
(oracle/_ref) and libmotif_b200.so into an executable.  Nothing is run (no
GPU needed)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers only in the build container")
def test_reference_binding_compiles_and_links(tmp_path):
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    snippet = re.search(r"```cpp\n(.*?)```", text, re.S).group(1)
    src = tmp_path / "b200.cpp"
    src.write_text(snippet + """
int main() {
  motif::DataGraph g = motif::DataGraph::from_edges(3, {{0, 1}, {1, 2}, {2, 0}});
  motif::QueryGraph q = motif::QueryGraph::from_edges(3, {{0, 1}, {1, 2}, {2, 0}});
  motif::Coloring chi = motif::random_coloring(g, 3, 7);
  return static_cast<int>(motif::count_colorful_b200(g, chi, q, motif::EngineKind::DB) > 6);
}
""")
    ref_lib = os.path.join(ROOT, "oracle", "_ref")
    lib = os.path.join(ROOT, "paper_1602_04478_b200")
    if not os.path.exists(os.path.join(ref_lib, "libmotif_ref.so")):
        pytest.skip("oracle/_ref not built")
    cmd = ["/usr/bin/g++", "-std=c++20", "-O0", "-I", REF_INC, "-I", os.path.join(ROOT, "include"), str(src),
           "-o", str(tmp_path / "b200"), "-L", ref_lib, "-lmotif_ref", "-L", lib, "-lmotif_b200", "-fopenmp",
           f"-Wl,-rpath,{ref_lib}:{lib}"]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    assert proc.returncode == 0, proc.stderr[-4000:]
