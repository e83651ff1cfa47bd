// Probe build of K2-TC: the product bp_tc.cu compiled with TF_TC_PROBE, so
// each role of bp_tc_kernel records its wait cycles per CTA (tile order
// index < 1024, first z-block) into a device buffer set with
// tf_bp_tc_probe().  Linked with the other csrc/*.cu into
// tools/micro/libtomofuse_probe.so by tools/tc_probe.py; never part of the
// product library (which has no global state).
#ifndef TF_TC_NOPROBE  // -DTF_TC_NOPROBE: the same experiment knobs, uninstrumented timing
#define TF_TC_PROBE 1
#endif
#ifdef TF_TC_SRC  // an alternative K2-TC source (A/B timing against an older revision)
#include TF_TC_SRC
#else
#include "../../paper_2505_13955_b200/csrc/bp_tc.cu"
#endif

extern "C" TF_API int tf_bp_tc_probe(void* buf) {
#ifdef TF_TC_PROBE
    tf::g_tc_probe = static_cast<long long*>(buf);
#else
    (void)buf;
#endif
    return TF_OK;
}
