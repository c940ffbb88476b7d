/* Device status block shared by the runtime library, every generated
 * mechanism TU and the Python ctypes mirror (paper_1905_02241_b200/runtime.py).
 *
 * The reference runtime raises InterpError for non-finite slots, Newton
 * non-convergence, the WHILE cap and singular pivots
 * (modlc/interp.py:285-286,406-411,538-545,619-622); the reference's emitted C
 * only counts `md->solver_failures` (modlc/codegen.py:239).  On the device
 * every failing lane proposes a lexicographic key (see nmodl::err_key); the
 * minimum survives, which is exactly the error the reference would raise
 * first.  Plain C so that the host header include/nmodl_b200.h can share it. */
#ifndef NMODL_B200_STATUS_H
#define NMODL_B200_STATUS_H

#define NMODL_NO_ERROR 0xffffffffffffffffull

typedef struct nmodl_status {
  unsigned long long err_key;     /* min error key, NMODL_NO_ERROR if none   */
  unsigned long long payload_key; /* key that owns `payload`                 */
  double payload;                 /* e.g. Newton residual of that instance   */
  int lock;                       /* spin lock guarding payload updates      */
  int reserved;
} nmodl_status;

#define NMODL_KIND_WHILE 0
#define NMODL_KIND_NEWTON 1
#define NMODL_KIND_SINGULAR 2

#endif
