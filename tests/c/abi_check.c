/* Plain C (C11) client of include/polyeval_b200.h: proves the boundary is a
 * C ABI (no C++ in the header) and exercises the host-only entry points —
 * program creation from terms and from a compiled program, introspection,
 * PTX generation and the ptxas build — without a GPU. Exit code 0 = pass. */
#include <stdio.h>
#include <string.h>

#include "polyeval_b200.h"

#define CHECK(x)                                                        \
  do {                                                                  \
    pe_status st_ = (x);                                                \
    if (st_ != PE_OK) {                                                 \
      fprintf(stderr, "%s -> %d: %s\n", #x, (int)st_, pe_last_error()); \
      return 1;                                                         \
    }                                                                   \
  } while (0)

int main(void) {
  /* 3x^8 - x^7 + 2x^6 + x^5 - 4x^4 + 9x^3 - 3x^2 - 2x + 1 (reference worked example) */
  const uint32_t exps[9] = {8, 7, 6, 5, 4, 3, 2, 1, 0};
  const double coefs[9] = {3, -1, 2, 1, -4, 9, -3, -2, 1};
  const pe_scheme_desc estrin = {PE_SCHEME_ESTRIN, 0, 0};
  pe_program* prog = NULL;
  CHECK(pe_program_create(exps, coefs, 9, 1, &estrin, PE_COEFF_F64, &prog));

  pe_program_info_t info;
  CHECK(pe_program_info(prog, &info));
  if (info.records != 9 || info.nvars != 1) return 2;

  size_t len = 0;
  CHECK(pe_program_ptx(prog, 0, NULL, 0, &len));
  if (len < 100) return 3;
  uint64_t cubin = 0;
  CHECK(pe_program_compile_only(prog, 3, &cubin)); /* interval kernel */
  if (cubin == 0) return 4;
  CHECK(pe_program_check_registers(prog));

  /* the same Hörner 3x^2 + 2x + 1 as a hand-flattened compiled program */
  const pe_record recs[3] = {
      {3.0, 0, -1, 0, 0, 0, 0, 0},
      {2.0, 0, -1, 0, 0, 0, 1, 0},
      {1.0, 0, -1, -1, 0, -1, 1, 0},
  };
  const uint32_t ends[1] = {1};
  const pe_compiled_program cp = {recs, 3, 1, 0, ends, 1};
  const uint32_t set0[1] = {1};
  const uint32_t* sets[1] = {set0};
  const size_t sizes[1] = {1};
  pe_program* imported = NULL;
  CHECK(pe_program_from_compiled(&cp, 1, 1, sets, sizes, PE_COEFF_F64, &imported));
  CHECK(pe_program_compile_only(imported, 0, &cubin));

  /* errors come back as status codes, never as exceptions */
  pe_program* bad = NULL;
  if (pe_program_create(exps, coefs, 9, 0, &estrin, PE_COEFF_F64, &bad) != PE_EINVAL) return 5;
  if (strlen(pe_last_error()) == 0) return 6;

  pe_program_destroy(imported);
  pe_program_destroy(prog);
  printf("%s: C ABI ok\n", pe_version());
  return 0;
}
