// ucac_part.h -- rank-local problem description of the bus-graph cut (partition.cu).
#pragma once
#include <cstdint>
#include <vector>

namespace ucac {

struct Halo {
    int nparts = 1, rank = 0;
    std::vector<int> own_bus, ghost_bus;       // global ids (local ids: own then ghost)
    std::vector<int> local_branch, phantom;    // global ids (local ids: local then phantom)
    std::vector<int> bus_local;                // global bus -> local id or -1
    std::vector<int> br_local;                 // global branch -> local id or -1
    std::vector<int> cut_local;                // local ids of my branches whose to-bus is remote
    std::vector<int> export_local;             // local ids of my buses that are a remote branch's to-bus
    std::vector<int> phantom_src;              // gathered-buffer slot (owner * max_cut + position)
    std::vector<int> ghost_src;                // gathered-buffer slot (owner * max_export + position)
    int max_cut = 0, max_export = 0;
};

int partition_buses(int nbus, int nbranch, const int32_t *from, const int32_t *to, const double *xy, int nparts,
                    int32_t *part, const double *branch_w);
Halo build_halo(int nbus, int nbranch, const int32_t *from, const int32_t *to, const int32_t *part, int nparts,
                int rank);

}  // namespace ucac
