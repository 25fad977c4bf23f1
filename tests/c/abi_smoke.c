/* Compiles include/gcb200.h as plain C11 and links libgcb200.so from C:
 * the drop-in boundary a non-Python host binds.  Calls
 * only entry points that need no GPU: the ABI version, the error string,
 * the launch counter, argument validation of a few entry points. */
#include <stdio.h>
#include <string.h>

#include "gcb200.h"

int main(void) {
    if (gc_abi_version() != GC_ABI_VERSION) {
        printf("abi mismatch %d != %d\n", gc_abi_version(), GC_ABI_VERSION);
        return 1;
    }
    gc_reset_launch_count();
    if (gc_launch_count() != 0) return 2;
    /* argument validation happens before any CUDA call */
    void* plan = 0;
    int rc = gc_plan_create(0, 0, 0, 0, 0, 0, &plan);
    if (rc != GC_ERR_CONFIG || plan != 0 || strlen(gc_last_error()) == 0) return 3;
    rc = gc_plan_run(0, 0, 0, 0);
    if (rc != GC_ERR_STATE) return 4;
    rc = gc_tier_compose(1, 0, 0, 0, 0, 0);
    if (rc != GC_ERR_CONFIG) return 5;
    printf("gcb200 C ABI %d ok: %s\n", gc_abi_version(), gc_last_error());
    return 0;
}
