"""Insert clock64 event stamps into k1w_stats_tc (wide.cuh) and a trace reader into smf.cu,
in place (debug aid)."""
import os
import sys

# Patches a COPY of the sources: usage `python <this> DIR` with DIR a directory holding a copy
# of paper_2003_02978_b200/ (e.g. made by `git archive HEAD paper_2003_02978_b200 include | tar
# -x -C DIR`); build it with `mkvariant.sh NAME DIR`. Refuses to touch the repository itself.
ROOT = os.path.abspath(sys.argv[1]) if len(sys.argv) > 1 else None
REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT is None or ROOT == REPO:
    raise SystemExit("usage: %s COPY_DIR (a copy of the sources, not the repository)" % sys.argv[0])
p = os.path.join(ROOT, "paper_2003_02978_b200/csrc/wide.cuh")
s = open(p).read()
s = s.replace("""constexpr int kTW = 13 * 32;""", """__device__ unsigned long long g_k1wtrace[2][8][256];
#define K1WTR(ev, i) do { if (blockIdx.y == 0 && blockIdx.x < 2 && (i) < 256) g_k1wtrace[blockIdx.x][ev][(i)] = clock64(); } while (0)
constexpr int kTW = 13 * 32;""", 1)
reps = [
    ("""            if (kb >= 2) mbar_wait(&op_empty[s2], ((kb >> 1) - 1) & 1);
            if (work) {
                const int p0 = kb * 32;
                // the extended-row entry""", """            if (tid == 0) K1WTR(0, kb);
            if (kb >= 2) mbar_wait(&op_empty[s2], ((kb >> 1) - 1) & 1);
            if (tid == 0) K1WTR(1, kb);
            if (work) {
                const int p0 = kb * 32;
                // the extended-row entry"""),
    ("""            if (lane == 0) mbar_arrive(&op_full[s2]);
        };""", """            if (lane == 0) mbar_arrive(&op_full[s2]);
            if (tid == 0) K1WTR(3, kb);
        };"""),
    ("""                mbar_wait(&op_full[s2], (kb >> 1) & 1);
                tc_fence_after();""", """                mbar_wait(&op_full[s2], (kb >> 1) & 1);
                K1WTR(4, kb);
                tc_fence_after();"""),
    ("""                mma_commit(&op_empty[s2]);""", """                mma_commit(&op_empty[s2]);
                K1WTR(5, kb);"""),
    ("""            mbar_wait(&acc_full[ab], (g >> 1) & 1);
            tc_fence_after();
            const uint32_t t0 = tmem + ((uint32_t)(32 * e) << 16) + (uint32_t)(ab * 256);""", """            mbar_wait(&acc_full[ab], (g >> 1) & 1);
            if (lane == 0 && e == 0) K1WTR(6, kb);
            tc_fence_after();
            const uint32_t t0 = tmem + ((uint32_t)(32 * e) << 16) + (uint32_t)(ab * 256);"""),
    ("""            if (lane == 0) mbar_arrive(&acc_empty[ab]);
            ++g;
            first = false;""", """            if (lane == 0) mbar_arrive(&acc_empty[ab]);
            if (lane == 0 && e == 0) K1WTR(7, kb);
            ++g;
            first = false;"""),
]
for a, b in reps:
    assert a in s, a[:60]
    s = s.replace(a, b, 1)
open(p, "w").write(s)
p = os.path.join(ROOT, "paper_2003_02978_b200/csrc/smf.cu")
s = open(p).read()
s += """
extern "C" int smf_debug_k1w_trace(unsigned long long* host, int n) {
    return (int)cudaMemcpyFromSymbol(host, smf::g_k1wtrace, sizeof(unsigned long long) * (size_t)n);
}
"""
open(p, "w").write(s)
