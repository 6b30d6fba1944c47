/* Stub libdw.so.1 for the Nsight Systems importer shipped inside this image's Nsight Compute
 * (QdstrmImporter -> libAnalysis.so needs libdw, which the image lacks). libdw is only used to
 * symbolise CPU backtraces; tools/nsys_run.sh captures with CPU sampling off (-s none), so every
 * entry point here just reports failure. Diagnostic tooling only — never linked by the product. */
#include <stddef.h>
void *dwarf_attr(void *d, unsigned n, void *r) { return NULL; }
void *dwarf_diecu(void *d, void *r, unsigned char *a, unsigned char *o) { return NULL; }
unsigned long dwarf_dieoffset(void *d) { return (unsigned long)-1; }
const char *dwarf_filesrc(void *f, size_t i, void *m, void *l) { return NULL; }
int dwarf_formudata(void *a, void *r) { return -1; }
int dwarf_getscopes(void *c, unsigned long pc, void **s) { return -1; }
int dwarf_getscopes_die(void *d, void **s) { return -1; }
int dwarf_getsrcfiles(void *c, void **f, size_t *n) { return -1; }
void *dwarf_offdie(void *d, unsigned long o, void *r) { return NULL; }
int dwarf_tag(void *d) { return -1; }
void *dwfl_addrmodule(void *d, unsigned long a) { return NULL; }
void *dwfl_begin(const void *cb) { return NULL; }
int dwfl_build_id_find_elf(void *m, void **u, const char *n, unsigned long b, char **f, void **e) { return -1; }
void dwfl_end(void *d) {}
void *dwfl_getsrc(void *d, unsigned long a) { return NULL; }
const char *dwfl_lineinfo(void *l, unsigned long *a, int *ln, int *c, void *m, void *e) { return NULL; }
void *dwfl_module_addrdie(void *m, unsigned long a, unsigned long *b) { return NULL; }
void *dwfl_module_getdwarf(void *m, unsigned long *b) { return NULL; }
void *dwfl_module_getsrc(void *m, unsigned long a) { return NULL; }
const char *dwfl_module_info(void *m, void ***u, unsigned long *s, unsigned long *e, unsigned long *db,
                             unsigned long *sb, const char **mf, const char **df) { return NULL; }
int dwfl_offline_section_address(void *m, void **u, const char *n, unsigned long b, const char *s,
                                 unsigned int sh, const void *shdr, unsigned long *a) { return -1; }
int dwfl_report_end(void *d, void *r, void *a) { return -1; }
void *dwfl_report_offline(void *d, const char *n, const char *f, int fd) { return NULL; }
int dwfl_standard_find_debuginfo(void *m, void **u, const char *n, unsigned long b, const char *f,
                                 const char *dl, unsigned int c, char **df) { return -1; }
