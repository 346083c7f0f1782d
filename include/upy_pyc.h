/*
 * upy_pyc.h -- C ABI of the native .pyc loader in libupy_cuda.so (host code).
 *
 * Replaces the reference's loader for the decompile path:
 *     unpyre.pyc.load_pyc(data) -> (VersionTag, CodeObject)
 *     (/root/reference/pkg/src/unpyre/pyc.py:50-52; parse_pyc_header :36-47,
 *      parse_marshal / _Reader / _read_code :78-352)
 * for a whole batch of files at once, producing the arena of include/upy.h.
 */
#ifndef UPY_PYC_H
#define UPY_PYC_H
#include "upy.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Host-side .pyc loader (≡ unpyre.pyc.load_pyc per file, pyc.py:36-52, with
 * parse_marshal :78-352): parses a batch of .pyc images (PEP 552 header +
 * marshal stream, CPython 3.8-3.11) straight into one arena image in host
 * memory, ready for a single H2D copy and upy_decompile_batch.  Files are
 * parsed on n_threads host threads (<= 0: all hardware threads).
 *
 * Per file: file_status is UPY_ST_OK or UPY_ST_UNKNOWN_MAGIC /
 * UPY_ST_TRUNCATED_HEADER / UPY_ST_MALFORMED_MARSHAL with the reference's
 * exception text in messages[msg_off .. +msg_len] and file_aux = the magic or
 * the byte offset; file_root is the file's index in the roots section (-1 on
 * error).  Section order: objs, consts, strs, refs, limbs, bytes, roots; the
 * device arena is {image + section_off[i], section_count[i]}. */
typedef struct {
  uint8_t*        image;              /* host arena image, sections 256-B aligned */
  uint64_t        image_bytes;
  uint64_t        section_off[7];
  int64_t         section_count[7];
  uint64_t        max_code_len, total_code_units;
  int64_t         n_files;
  const int32_t*  file_status;
  const int32_t*  file_root;
  const int64_t*  file_aux;
  const char*     messages;
  const uint64_t* msg_off;
  const uint32_t* msg_len;
} upy_pyc_batch;

/* flags for upy_pyc_load */
enum { UPY_PYC_DEFER_IMAGE = 1 };  /* parse and lay out only: image == NULL, image_bytes set; the
                                      caller then fills its own buffer (e.g. reusable page-locked
                                      memory for a direct H2D DMA) with upy_pyc_write_image */

/* Returns 0 on success (per-file failures are in the batch), 1 on bad arguments, 2 when
 * the image cannot be allocated. */
int upy_pyc_load(const uint8_t* const* data, const uint64_t* sizes, int64_t n_files, int n_threads,
                 int flags, upy_pyc_batch** out);
/* Write the arena image of a batch into dst (dst_bytes >= image_bytes).  0 on success. */
int upy_pyc_write_image(upy_pyc_batch* batch, uint8_t* dst, uint64_t dst_bytes);
void upy_pyc_free(upy_pyc_batch* batch);

#ifdef __cplusplus
}
#endif
#endif
