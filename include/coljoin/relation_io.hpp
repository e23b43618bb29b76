// Relation manifest I/O (reference: include/coljoin/relation_io.hpp:7-15,
// src/relation_io.cpp:48-103) — the on-disk exchange format that feeds the
// same inputs to the reference's CPU engine and to this library.
//
// Layout of a relation directory: `manifest.txt` (one field per line:
// `name <n>`, `rows <n>`, `key_unique <0|1>`, then `column <name> <u32|u64>
// <file>` for the key and every payload in order) and one raw little-endian
// file per column.  Implemented in paper_2312_00720_b200/host/io.cpp; the
// Python mirror (coljoin.export_relation / import_relation) reads and writes
// the same directories straight from / into device columns.
#pragma once

#include <filesystem>

#include "coljoin/column.hpp"

namespace coljoin::workloads {

/// Writes manifest.txt plus key.bin, payload0.bin, ... into dir (created).
void export_relation(const Relation& rel, const std::filesystem::path& dir);

/// Reads a directory written by export_relation (this library's or the
/// reference's).  SchemaError on a missing/malformed manifest or short file.
Relation import_relation(const std::filesystem::path& dir);

}  // namespace coljoin::workloads
