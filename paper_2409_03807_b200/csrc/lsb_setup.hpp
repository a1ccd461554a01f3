// Host-side setup (kernel K0 of SURVEY §2.2): procedural meshes, rest-state
// precompute, lumped mass, vertex->element CSR and decoder initialisation.
// Runs once per problem on the host in fp64; results are uploaded to HBM.
#pragma once

#include <cstdint>
#include <random>
#include <string>
#include <vector>

namespace lsb {

// Bit-stable RNG helpers with the reference's semantics
// (proj/include/lipsub/rng.hpp:11-51).
using Rng = std::mt19937_64;
double randu(Rng& rng);
double randn(Rng& rng);
Rng substream(std::uint64_t seed, std::uint64_t tag);

struct HostMesh {
    int V = 0, E = 0;
    std::vector<double> X;      // V*3
    std::vector<int> T;         // E*4
    std::vector<int> pinned;    // sorted unique
    // derived by precompute():
    std::vector<double> Dminv;  // E*9 row-major
    std::vector<double> vol;    // E
    std::vector<int> free_index;  // V (slot or -1)
    std::vector<int> free_vertex; // n_free (vertex id of slot)
    int n_free = 0;
    // vertex(free slot) -> incident (tet*4 + local slot), ascending tet id
    std::vector<int> csr_ptr, csr_ent;
};

// Validates and precomputes (build_mesh semantics, proj/src/mesh.cpp:90-145):
// out-of-range ids and det Dm <= 1e-14 throw std::runtime_error.
void precompute(HostMesh& m);

// Six-tet (Kuhn) bar: vertex id (i*vy+j)*vz+k, coordinates (w i/nx, h j/ny, d k/nz)
// (mesh.cpp:357-364), optional Gaussian jitter (sigma = jitter_frac * cell,
// substream(seed, 1), vertex order), orientation fix (mesh.cpp:386-391), pins
// on the i == 0 face (mesh.cpp:392-395).
HostMesh make_bar_mesh(int nx, int ny, int nz, double w, double h, double d, double jitter_frac,
                       std::uint64_t seed, bool pin_left);

// Lumped vertex mass (mesh.cpp:417-434) per free DOF.
std::vector<double> lump_mass(const HostMesh& m, double density, double* total);

struct HostLayer {
    int rows = 0, cols = 0, act = 0;
    std::vector<double> W;  // row-major
    std::vector<double> b;
};
struct HostDecoder {
    int r = 0, n = 0;
    std::vector<HostLayer> layers;
    std::vector<double> shift, scale;
};

// Xavier-normal MLP (BASELINE.json): make_mlp_model's structure
// (net.cpp:90-123) with std sqrt(2/(fan_in+fan_out)), randn from
// substream(seed, 0), column-major fill; output layer drawn 3V x width and
// pinned rows dropped; shift = rest free DOFs, scale = out_scale.
HostDecoder make_bar_decoder(const HostMesh& m, int r, int hidden_layers, int width, int act,
                             std::uint64_t seed, double out_scale);

}  // namespace lsb
