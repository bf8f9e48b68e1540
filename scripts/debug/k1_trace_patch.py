"""Insert clock64 event stamps into k1_stats_tc (kernels.cuh) and a trace reader into smf.cu,
in place (debug aid).
Events per tile i of CTA 0 (group leaders: lane 0 of warps 0 and 4):
0 raw ready, 1 sigma dot done, 2 operand stage free, 3 stores issued, 4 published,
5 MMA start, 6 MMA issued, 7 TMA issue."""
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
s = s.replace("""constexpr int kFlushTC = SMF_K1TC_FLUSH;""", """constexpr int kFlushTC = SMF_K1TC_FLUSH;
__device__ unsigned long long g_k1trace[10][4096];
#define K1TR(ev, i) do { if (blockIdx.x == 0 && (i) < 4096) g_k1trace[ev][(i)] = clock64(); } while (0)
//""", 1)
reps = [
    ("""            mbar_wait(&raw_full[s], (i / K::RS) & 1);
            if (SMF_K1TC_EXP & 8) {""", """            mbar_wait(&raw_full[s], (i / K::RS) & 1);
            if (lane == 0 && (wid & 3) == 0) K1TR(0, i);
            if (SMF_K1TC_EXP & 8) {"""),
    ("""            sg += __shfl_xor_sync(0xffffffffu, sg, 16);""", """            sg += __shfl_xor_sync(0xffffffffu, sg, 16);
            if (lane == 0 && (wid & 3) == 0 && sg != 1.2345e30f) K1TR(1, i);"""),
    ("""            if (i >= kOpStagesTC) mbar_wait(&op_empty[o], ((i / kOpStagesTC) - 1) & 1);
            const uint32_t ob = ops0 + o * K::OPSTAGE;""", """            if (i >= kOpStagesTC) mbar_wait(&op_empty[o], ((i / kOpStagesTC) - 1) & 1);
            if (lane == 0 && (wid & 3) == 0) K1TR(2, i);
            const uint32_t ob = ops0 + o * K::OPSTAGE;"""),
    ("""            fence_proxy_async();   // generic-proxy smem writes -> visible to the tensor core
            __syncwarp();
            if (lane == 0) mbar_arrive(&op_full[o]);""", """            if (lane == 0 && (wid & 3) == 0) K1TR(3, i);
            fence_proxy_async();   // generic-proxy smem writes -> visible to the tensor core
            __syncwarp();
            if (lane == 0) mbar_arrive(&op_full[o]);
            if (lane == 0 && (wid & 3) == 0) K1TR(4, i);"""),
    ("""                mbar_wait(&op_full[o], (i / kOpStagesTC) & 1);""", """                mbar_wait(&op_full[o], (i / kOpStagesTC) & 1);
                K1TR(5, i);"""),
    ("""                mma_commit(&op_empty[o]);""", """                mma_commit(&op_empty[o]);
                K1TR(6, i);"""),
    ("""                mbar_arrive_expect_tx(&raw_full[s], Raw::TX);""", """                mbar_arrive_expect_tx(&raw_full[s], Raw::TX);
                K1TR(7, i);"""),
    ("""            mbar_wait(&acc_full[ab], (g >> 1) & 1);
            tc_fence_after();
            const uint32_t t0 = tmem + ((uint32_t)(32 * e) << 16) + (uint32_t)(ab * K::NCOL);""", """            mbar_wait(&acc_full[ab], (g >> 1) & 1);
            if (lane == 0 && e == 0) K1TR(8, i);
            tc_fence_after();
            const uint32_t t0 = tmem + ((uint32_t)(32 * e) << 16) + (uint32_t)(ab * K::NCOL);"""),
    ("""            if (lane == 0) mbar_arrive(&acc_empty[ab]);
            ++g;
            if (col_end && live) {""", """            if (lane == 0) mbar_arrive(&acc_empty[ab]);
            if (lane == 0 && e == 0) K1TR(9, i);
            ++g;
            if (col_end && live) {"""),
]
for a, b in reps:
    assert a in s, a[:70]
    s = s.replace(a, b, 1)
open(p, "w").write(s)
p = os.path.join(ROOT, "paper_2003_02978_b200/csrc/smf.cu")
s = open(p).read()
s += """
extern "C" int smf_debug_k1_trace(unsigned long long* host, int n) {
    return (int)cudaMemcpyFromSymbol(host, smf::g_k1trace, sizeof(unsigned long long) * (size_t)n);
}
"""
open(p, "w").write(s)
