/*
 * sst_host.h -- host-side utilities of libsst_gpu.so (no device work): meshes,
 * SDF cache files and PFM output, C ABI mirrors of the reference's host
 * functions so that callers can build scenes without the reference library.
 * Return codes as in sst_gpu.h; messages via sst_gpu_last_error().
 */
#ifndef SST_HOST_H
#define SST_HOST_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* make_icosphere (mesh.hpp:46-48, mesh.cpp:154-185): identical vertex/face
 * order. Buffers are allocated by the library; free with sst_mesh_free. */
int sst_mesh_icosphere(int subdivisions, double radius, double** positions, uint32_t* n_vertices,
                       uint32_t** triangles, uint32_t* n_triangles);
/* make_bumpy_sphere (mesh.hpp:50-53, mesh.cpp:187-197). */
int sst_mesh_bumpy_sphere(int subdivisions, double radius, double amplitude, double frequency,
                          double** positions, uint32_t* n_vertices, uint32_t** triangles,
                          uint32_t* n_triangles);
/* load_obj (mesh.hpp:37-43, mesh.cpp:77-122): v/f records, fan triangulation,
 * negative indices, degenerate faces dropped and counted. */
int sst_mesh_load_obj(const char* path, double scale, double** positions, uint32_t* n_vertices,
                      uint32_t** triangles, uint32_t* n_triangles, uint64_t* dropped_degenerate);
void sst_mesh_free(double* positions, uint32_t* triangles);

/* SSDF cache files (sdf.cpp:71-101). */
int sst_sdf_save(const char* path, const double origin[3], double voxel, const uint32_t dims[3],
                 const float* values, uint64_t mesh_fingerprint);
int sst_sdf_load(const char* path, double origin[3], double* voxel, uint32_t dims[3],
                 float** values, uint64_t* mesh_fingerprint);
void sst_sdf_free(float* values);

/* save_dataset (dataset.cpp:94-119): SSWK v1, little-endian, 52-byte records
 * (sst_training_sample from sst_gpu.h). phi_kind/phi_a/phi_b as PhiSampler. */
int sst_dataset_save(const char* path, uint64_t count, float sigma_t_lo, float sigma_t_hi, float g_lo,
                     float g_hi, uint32_t phi_kind, float phi_a, float phi_b, uint64_t seed,
                     const void* samples);

/* DatasetHeader (dataset.hpp:43-50) as stored in an SSWK file. */
typedef struct sst_dataset_header {
    uint32_t version;
    uint64_t count;
    float sigma_t_lo, sigma_t_hi, g_lo, g_hi;
    uint32_t phi_kind; /* PhiSampler::Kind */
    float phi_a, phi_b;
    uint64_t seed;
} sst_dataset_header;

/* load_dataset (dataset.cpp:121-151): SSWK v1. Call with samples == NULL to read the
 * header (count) only, then with a buffer of >= header->count 52-byte records
 * (capacity = records it holds). Errors as the reference's (SST_E_RUNTIME): missing
 * file, "dataset <path>: bad magic bytes", "...: unsupported version",
 * "...: truncated or corrupt file"; capacity < count is SST_E_INVALID_ARGUMENT. */
int sst_dataset_load(const char* path, sst_dataset_header* header, void* samples, uint64_t capacity);

/* export_dataset_csv (dataset.cpp:153-164): header line + one "%.9g" row per record. */
int sst_dataset_export_csv(const char* path, uint64_t count, const void* samples);

/* save_pfm (image.cpp:32-41): little-endian "PF", bottom row first. */
int sst_image_save_pfm(const char* path, uint32_t width, uint32_t height, const float* rgb);

/* save_pfm_gray (image.cpp:62-73): one-channel "Pf", bottom row first. */
int sst_image_save_pfm_gray(const char* path, uint32_t width, uint32_t height, const float* values);

/* load_pfm (image.cpp:43-60): little-endian colour PFM only (the reference's errors:
 * "not a color PFM file", "big-endian PFM unsupported", "truncated PFM" -> SST_E_RUNTIME).
 * rgb == NULL queries width/height only; otherwise capacity (floats) must be >= w*h*3. */
int sst_image_load_pfm(const char* path, uint32_t* width, uint32_t* height, float* rgb,
                       uint64_t capacity);

/* save_png (image.cpp:101-138): 8-bit sRGB truecolor, clamp to [0,1], lround, filter 0,
 * zlib level 9 single IDAT; byte-identical to the reference with the same zlib. */
int sst_image_save_png(const char* path, uint32_t width, uint32_t height, const float* rgb);

#ifdef __cplusplus
}
#endif
#endif
