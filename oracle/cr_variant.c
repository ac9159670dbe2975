/* Experiment build (test infrastructure, tools/crlibm_decisions.py): the
 * oracle with glibc's sin/cos/acos/asin/atan2/hypot replaced by the
 * correctly rounded restatement the device's literal solver uses
 * (sd_crlibm.h).  Comparing it with the glibc oracle measures how often the
 * reference's decisions and values depend on glibc's misrounded last bits. */
#include "../paper_1306_6291_b200/csrc/sd_crlibm.h"
#define sin sdcr_sin
#define cos sdcr_cos
#define acos sdcr_acos
#define asin sdcr_asin
#define atan2 sdcr_atan2
#define hypot sdcr_hypot
#define sincos sdcr_sincos
#include "symdiag_oracle.c"
