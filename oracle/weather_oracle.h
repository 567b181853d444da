/* oracle/weather_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference minimal-weather hot path
 * (/root/reference/proj/src/weather.cpp).  Used by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg as the CHECKER; the product path never links
 * or calls it.  Parity of this restatement is pinned against the compiled
 * reference (oracle/_ref) and the committed golden fixtures (tests/golden/).
 *
 * Buffers are logical column-major with the reference's inclusive bounds:
 * 3D fields (0..nx+1, 0..ny+1, 1..nz), 2D fields (0..nx+1, 0..ny+1)
 * (weather.cpp:71,77).
 */
#ifndef HFT_WEATHER_ORACLE_H
#define HFT_WEATHER_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct wo_grid { /* field order mirrors hft::GridConfig, weather.hpp:27-34 */
    int64_t nx, ny, nz;
    double timestep, output_timestep, diffusion_velocity, radiation_intensity,
        transfer_velocity, surf_energy, pbl_energy;
} wo_grid;

int wo_validate(const wo_grid* g, char* msg, size_t cap);
void wo_init(const wo_grid* g, double* e, double* eu, double* sf, double* pb);
void wo_step(const wo_grid* g, double* e, double* eu, const double* sf, const double* pb);
void wo_steps(const wo_grid* g, int64_t steps, double* e, double* eu, const double* sf,
              const double* pb);
void wo_physics(const wo_grid* g, double* e, const double* sf, const double* pb);
void wo_diffuse(const wo_grid* g, const double* e, double* u);
int wo_compare_arrays(size_t n, const double* a, const double* b, double* max_abs,
                      double* nrmse, size_t* worst);
void wo_unpermute(int rank, const int64_t* lo, const int64_t* hi, const int* order,
                  const double* raw, double* out);
uint64_t wo_fnv1a64(const double* a, size_t n);

#ifdef __cplusplus
}
#endif
#endif
