// Relation manifests — the reference's on-disk exchange format
// (interface: include/coljoin/relation_io.hpp:7-15, format:
// src/relation_io.cpp:48-103), so the same inputs feed the reference's CPU
// engine and this library.
//
// A relation directory holds `manifest.txt`, one field per line:
//     name <name>
//     rows <n>
//     key_unique <0|1>
//     column key <u32|u64> key.bin
//     column payload<c> <u32|u64> payload<c>.bin      (one line per payload)
// and one raw little-endian file per column.  C++: implemented in
// paper_2312_00720_b200/host/io.cpp; Python: paper_2312_00720_b200.
// export_relation / import_relation (import straight into device columns).
#pragma once

#include <filesystem>

#include "coljoin/column.hpp"

namespace coljoin::workloads {

// Creates `dir` if needed and writes the manifest plus key.bin, payload0.bin, ...
void export_relation(const Relation& relation, const std::filesystem::path& dir);

// Reads a directory written by export_relation (ours or the reference's);
// SchemaError on a missing or malformed manifest or a short column file.
Relation import_relation(const std::filesystem::path& dir);

}  // namespace coljoin::workloads
