/*
 * favest_io.h -- host codecs for the reference's file formats, in the same
 * library as the transforms (libfavest_b200.so).
 *
 * Replaces the formatting / parsing loops of favest/io.py (format_float
 * :30-31, write_rule_file :33-38, write_coefficients :62-77,
 * read_coefficients :80-95, write_samples :98-108, read_samples :111-133,
 * write_csv :136-145) and favest/quadrature.py:_read_columns (:112-131).
 * The calls work on memory buffers; the caller opens, reads and writes the
 * file.  Output bytes equal the reference writers' (17 significant digits,
 * Python's "nan"/"inf" spellings, csv "\r\n" rows); parsing follows Python's
 * float() grammar and json.load's syntax, and yields bit-identical doubles.
 *
 * Buffers returned through char** / double** are malloc'd: release them with
 * fv_io_free.  Status codes as in favest_b200.h plus FV_ETYPE (the
 * reference raises TypeError).  Error messages carry "{path}" where the
 * reference prints the file name.
 */
#ifndef FAVEST_IO_H
#define FAVEST_IO_H

#ifdef __cplusplus
extern "C" {
#endif

#define FV_ETYPE 6

void fv_io_free(void* p);

/* Rows of doubles [nrows][ncols] as text, every value format(x, ".17g"):
 * sep ' ' with "\n" rows (rule files) or ',' with "\r\n" rows (csv.writer).
 * Appends to the malloc'd buffer *out of *len bytes (NULL / 0 to start one). */
int fv_io_format_table(const double* data, long long nrows, int ncols, int sep, int crlf, char** out, long long* len);

/* The coefficient file of write_coefficients: a, b complex128 [(lmax+1)^2]. */
int fv_io_format_coefficients(int lmax, const double* a, const double* b, char** out, long long* len);

/* Parse a column file: mode 0 = rule / design file (_read_columns), mode 1 =
 * sample CSV (read_samples, 8 columns).  *data = [nrows][ncols] doubles. */
int fv_io_parse_columns(const char* text, long long n, int mode, double** data, long long* nrows, int* ncols);

/* Parse a coefficient file: *lmax and complex128 arrays *a, *b of (lmax+1)^2. */
int fv_io_parse_coefficients(const char* text, long long n, int* lmax, double** a, double** b);

#ifdef __cplusplus
}
#endif

#endif /* FAVEST_IO_H */
