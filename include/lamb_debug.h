/*
 * lamb_debug.h — exported ONLY by liblamb_debug.so (the -DLAMB_DEBUG build; paper_2402_15627_b200/
 * build.py --debug).  Test hooks for the device-side checks that stand in for compute-sanitizer
 * (closed on this GPU pool): they corrupt internal state on purpose so a test can see a check fire.
 * Not part of the product ABI (include/lamb.h); liblamb.so does not export them.
 */
#ifndef LAMB_DEBUG_H_
#define LAMB_DEBUG_H_

#include <stdint.h>

#include "lamb.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Overwrites the flat offset of work item `item` of handle `h` (device table) with `flat_off`:
 * the next step's pass kernels must stop with a "LAMB_DEBUG" bounds/alignment message and a
 * trap instead of reading or writing outside the buffers.  Synchronous.  EINVAL: item out of
 * range. */
lamb_status lamb_debug_corrupt_item(lamb_t h, int64_t item, int64_t flat_off);

#ifdef __cplusplus
}
#endif
#endif /* LAMB_DEBUG_H_ */
