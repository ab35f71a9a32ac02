#!/bin/bash
# Writes profiles/r02_sass_execute_kernel.txt: the SASS of execute_kernel<EXACT=0, FINE=1, DBG=0> (the kernel the
# bench times) from the built library, with a count of the instruction mnemonics that matter on sm_100a.
set -e
cd "$(dirname "$0")/.."
LIB=paper_1203_1692_b200/csrc/libspamm_b200.so
OUT=profiles/r02_sass_execute_kernel.txt
FN='_Z14execute_kernelILb0ELb1ELb0EEv8ExecArgs'
TMP=$(mktemp)
cuobjdump -sass -fun "$FN" "$LIB" > "$TMP"
{
  echo "# SASS of execute_kernel<EXACT=false, FINE=true, DBG=false> (sm_100a), cuobjdump -sass -fun $FN $LIB"
  echo "# regenerate: bash profiles/sass_listing.sh"
  echo "#"
  echo "# mnemonic counts (static):"
  for m in FFMA2 FFMA FMUL2 FMUL DFMA DMUL DSETP LDS.128 LDS STS LDG STG UBLKCP SYNCS.ARRIVE SYNCS.PHASECHK ATOMG ATOM RED \
           SHFL VOTE BAR NANOSLEEP ACQBULK UTMALDG UTCMMA UTCHMMA UTCBAR TCGEN05 LDTM STTM HMMA QGMMA; do
    c=$(grep -c -E "^\s+/\*[0-9a-f]+\*/\s+(@!?U?P[0-9T]+\s+)?${m//./\\.}[ .;]" "$TMP" || true)
    printf "#   %-16s %6d\n" "$m" "$c"
  done
  echo "#"
  echo "# present: UBLKCP (cp.async.bulk global->shared), SYNCS.* (mbarrier arrive/expect_tx/try_wait), FFMA2 (packed FP32 FMA),"
  echo "#          ACQBULK/griddepcontrol (programmatic dependent launch).  absent: UTCMMA/tcgen05.*, UTMALDG (tensor-map TMA),"
  echo "#          LDTM/STTM (tensor memory), HMMA: the products are FP32 SIMT by design (DESIGN.md, numeric kernel)."
  echo "#"
  cat "$TMP"
} > "$OUT"
rm -f "$TMP"
grep "^#" "$OUT"
