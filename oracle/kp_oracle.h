/* ORACLE — TEST INFRASTRUCTURE ONLY (see kp_oracle.cpp header).
 * Shares only the plain struct layouts of the public ABI header. */
#ifndef KP_ORACLE_H
#define KP_ORACLE_H
#include "../include/kronprec_b200.h"
#endif
