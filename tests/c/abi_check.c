/* The drop-in boundary from plain C (no C++ anywhere in this translation unit): both public
 * headers compile as pedantic C99 and link against the two shipped libraries.  With a GPU the
 * program creates an engine and moves one node host -> HBM -> host (K1 + K2) through the
 * C-ABI, checking the bytes; without one it checks the documented no-fallback failure.
 * Built and run by tests/test_c_abi.py. */
#include <stdio.h>
#include <string.h>

#include "kvflow.h"
#include "kvflow_host.h"

int main(void) {
    kvf_geometry g = {2, 8, 8, 0, 128, 2};
    kvf_engine_config c;
    kvf_engine* e = NULL;
    kvf_run h = {0, 64}, d = {0, 64}, h2 = {64, 64};
    uint64_t cids[64], a = 0, b = 0;
    unsigned i;
    int rc;
    memset(&c, 0, sizeof c);
    c.device = 0;
    c.gpu_slots = 256;
    c.host_slots = 256;
    c.pcie_mode = KVF_COPY_SM_VEC;
    c.host_numa_node = -1;
    rc = kvf_engine_create(&g, &c, &e);
    if (rc == KVF_E_NO_DEVICE) {
        printf("no-device %d: %s\n", rc, kvf_last_error());
        return 0;
    }
    if (rc != KVF_OK) {
        printf("create failed %d: %s\n", rc, kvf_last_error());
        return 1;
    }
    for (i = 0; i < 64; ++i) cids[i] = 0x9e3779b97f4a7c15ull * (i + 1);
    rc = kvf_fill_payload(e, KVF_TIER_HOST, &h, 1, cids, 64);
    if (!rc) rc = kvf_h2d_gather(e, 1, &h, 1, &d, 1);  /* K1 */
    if (!rc) rc = kvf_job_wait(e, 1);
    if (!rc) rc = kvf_job_release(e, 1);
    if (!rc) rc = kvf_d2h_scatter(e, 2, &d, 1, &h2, 1);  /* K2 */
    if (!rc) rc = kvf_job_wait(e, 2);
    if (!rc) rc = kvf_job_release(e, 2);
    if (!rc) rc = kvf_checksum(e, KVF_TIER_HOST, &h2, 1, &a);
    if (!rc) rc = kvf_payload_checksum(e, cids, 64, &b);
    if (rc) printf("failed %d: %s\n", rc, kvf_last_error());
    else printf("round trip %s\n", a == b ? "ok" : "MISMATCH");
    kvf_engine_destroy(e);
    return rc || a != b;
}
