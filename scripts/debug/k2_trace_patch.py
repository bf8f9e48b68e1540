"""Insert clock64 phase stamps into k2_update (kernels.cuh) and a reader into smf.cu, in place
(debug aid)."""
import os
import sys

# Patches a COPY of the sources: usage `python <this> DIR` with DIR a directory holding a copy
# of paper_2003_02978_b200/ (e.g. made by `git archive HEAD paper_2003_02978_b200 include | tar
# -x -C DIR`); build it with `mkvariant.sh NAME DIR`. Refuses to touch the repository itself.
ROOT = os.path.abspath(sys.argv[1]) if len(sys.argv) > 1 else None
REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT is None or ROOT == REPO:
    raise SystemExit("usage: %s COPY_DIR (a copy of the sources, not the repository)" % sys.argv[0])
p = os.path.join(ROOT, "paper_2003_02978_b200/csrc/kernels.cuh")
s = open(p).read()
s = s.replace("__global__ void __launch_bounds__(128, 5) k2_update(UpdateArgs a) {",
              "__device__ unsigned long long g_k2trace[64][8];\n"
              "#define K2TR(ev) do { if (threadIdx.x == 0 && blockIdx.x < 64) g_k2trace[blockIdx.x][ev] = clock64(); } while (0)\n"
              "__global__ void __launch_bounds__(128, 5) k2_update(UpdateArgs a) {", 1)
reps = [
    ("""    if (st0 != COL_OK) return;   // uniform per block""", """    if (st0 != COL_OK) return;   // uniform per block
    K2TR(0);"""),
    ("""    const double invN = 1.0 / nvc;""", """    K2TR(1);
    const double invN = 1.0 / nvc;"""),
    ("""    // 2. y_t = A^-1 t, y_h = A^-1 h  (A^-1 symmetric: row i, column = tid -> coalesced)""",
     """    K2TR(2);
    // 2. y_t = A^-1 t, y_h = A^-1 h  (A^-1 symmetric: row i, column = tid -> coalesced)"""),
    ("""    // 3. G_ij = u_i . y_j""", """    K2TR(3);
    // 3. G_ij = u_i . y_j"""),
    ("""    // 4. z = y_t - Y M (I + G M)^-1 U^T A^-1 t   (Woodbury)""", """    K2TR(4);
    // 4. z = y_t - Y M (I + G M)^-1 U^T A^-1 t   (Woodbury)"""),
    ("""    block_sum<3>(qc, scratch);
    int st = sh_st;""", """    block_sum<3>(qc, scratch);
    K2TR(5);
    int st = sh_st;"""),
]
for a, b in reps:
    assert a in s, a[:60]
    s = s.replace(a, b, 1)
open(p, "w").write(s)
p = os.path.join(ROOT, "paper_2003_02978_b200/csrc/smf.cu")
s = open(p).read()
s += """
extern "C" int smf_debug_k2_trace(unsigned long long* host, int n) {
    return (int)cudaMemcpyFromSymbol(host, smf::g_k2trace, sizeof(unsigned long long) * (size_t)n);
}
"""
open(p, "w").write(s)
